"""SPEC.md's SparseUpdate wire format (SPEC.md:131 word layout, :202 header)
at the C ABI: gtc_wire_pack / gtc_wire_unpack convert between the hot path's
canonical words (index << 1 | neg, R3) and SPEC's interchange layout
(bit 31 = sign, bits 0..30 = index).  Host-only calls: no GPU needed."""
import struct

import numpy as np
import pytest

import paper_1904_10584_b200 as gtc


def canon(i, neg):
    return (i << 1) | int(neg)


def spec_words(blob):
    k = struct.unpack_from("<I", blob, 16)[0]
    return list(struct.unpack_from(f"<{k}I", blob, 20))


def test_spec_pack_word_examples():
    # (5, negative) -> 0x80000005; (0, positive) -> 0x00000000
    blob = gtc.gtc_wire_pack(np.array([canon(0, False), canon(5, True)], np.uint32), 8, 8.0)
    assert spec_words(blob) == [0x00000000, 0x80000005]


def test_header_layout():
    # little-endian magic "GTCU", dim (u64), tau (f32), word count (u32), words
    words = np.array([canon(1, True), canon(2, False), canon(1000, True)], np.uint32)
    blob = gtc.gtc_wire_pack(words, 4097, 0.5)
    assert blob[:4] == b"GTCU"
    assert struct.unpack_from("<Q", blob, 4)[0] == 4097
    assert struct.unpack_from("<f", blob, 12)[0] == 0.5
    assert struct.unpack_from("<I", blob, 16)[0] == 3
    assert len(blob) == 20 + 4 * 3  # 4 x word count + a fixed header
    assert spec_words(blob) == [0x80000001, 0x00000002, 0x800003E8]


def test_worked_vector_through_the_oracle():
    # v = [3, -10, 20, 8], tau = 8 -> words for (idx 1, -), (idx 2, +)
    import oracle

    g = np.array([3.0, -10.0, 20.0, 8.0], np.float32)
    r = np.zeros(4, np.float32)
    words, _ = oracle.encode(g, r, 8.0, oracle.CMP_GT)
    blob = gtc.gtc_wire_pack(words, 4, 8.0)
    assert spec_words(blob) == [0x80000001, 0x00000002]
    back, dim, tau = gtc.gtc_wire_unpack(blob)
    assert np.array_equal(back, words) and dim == 4 and tau == 8.0


def test_roundtrip_random():
    # exhaustive roundtrip over 1e5 random indices
    rng = np.random.default_rng(1904)
    dim = (1 << 31) - 1
    idx = np.unique(rng.integers(0, dim, 100_000, dtype=np.int64))
    neg = rng.integers(0, 2, idx.size)
    words = ((idx << 1) | neg).astype(np.uint32)
    blob = gtc.gtc_wire_pack(words, dim, 8.0)
    sw = np.frombuffer(blob, dtype="<u4", offset=20)
    assert np.array_equal(sw & 0x7FFFFFFF, idx) and np.array_equal(sw >> 31, neg)
    back, d, t = gtc.gtc_wire_unpack(blob)
    assert np.array_equal(back, words) and d == dim and t == 8.0


def test_empty_update():
    blob = gtc.gtc_wire_pack(np.zeros(0, np.uint32), 4, 8.0)
    assert len(blob) == 20
    back, dim, tau = gtc.gtc_wire_unpack(blob)
    assert back.size == 0 and dim == 4


@pytest.mark.parametrize("words,dim,status", [
    ([canon(3, 0), canon(3, 1)], 8, gtc.GTC_ECORRUPT),   # not strictly ascending
    ([canon(5, 0), canon(2, 0)], 8, gtc.GTC_ECORRUPT),   # descending
    ([canon(8, 0)], 8, gtc.GTC_ECORRUPT),                # index >= dim
    ([], 1 << 31, gtc.GTC_EDIM),                         # dim beyond the 31-bit index field
])
def test_pack_rejects(words, dim, status):
    with pytest.raises(gtc.GTCError) as e:
        gtc.gtc_wire_pack(np.array(words, np.uint32), dim, 8.0)
    assert e.value.status == status


def test_unpack_rejects():
    good = gtc.gtc_wire_pack(np.array([canon(1, 0), canon(4, 1)], np.uint32), 8, 8.0)
    bad = [b"GTCV" + good[4:],                                   # magic
           good[:-4],                                            # truncated
           good[:20] + struct.pack("<II", 0x80000004, 0x00000001),  # not ascending
           good[:4] + struct.pack("<Q", 4) + good[12:],          # index 4 >= dim 4
           good[:12] + struct.pack("<f", -1.0) + good[16:]]      # tau <= 0
    for b in bad:
        with pytest.raises(gtc.GTCError) as e:
            gtc.gtc_wire_unpack(b)
        assert e.value.status == gtc.GTC_ECORRUPT
