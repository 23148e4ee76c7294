"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/gtc.h declares; the binding marshals every one of them."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("gtc.h", "bmuf.h")]


def declared_functions():
    names = set()
    for h in HEADERS:
        src = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        names |= set(re.findall(r"\b((?:gtc|bmuf)_[a-z_]+)\s*\(", src))
    return sorted(names)


def test_header_declares_the_boundary():
    fns = declared_functions()
    for name in ("gtc_init", "gtc_encode", "gtc_exchange", "gtc_decode_apply", "gtc_destroy", "bmuf_sync"):
        assert name in fns


def test_library_loads_and_exports_every_symbol():
    import paper_1904_10584_b200 as gtc
    from paper_1904_10584_b200 import _build

    _build.build()
    lib = gtc.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in gtc._SIGS, f"binding lacks {name}"
        assert callable(getattr(gtc, name)), f"binding lacks python {name}"
    out = subprocess.run(["nm", "-D", "--defined-only", gtc.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_host_side_validation_without_gpu():
    """Argument checks that need no device."""
    import paper_1904_10584_b200 as gtc

    with pytest.raises(gtc.GTCError) as e:
        gtc.gtc_init(1 << 31, 8.0)
    assert e.value.status == gtc.GTC_EDIM
    for bad in (0.0, -1.0, float("nan"), float("inf")):
        with pytest.raises(gtc.GTCError) as e:
            gtc.gtc_init(10, bad)
        assert e.value.status == gtc.GTC_EINVAL
    with pytest.raises(gtc.GTCError):
        gtc.gtc_init(10, 8.0, rank=1, world=1)
    with pytest.raises(gtc.GTCError):
        gtc.gtc_init(10, 8.0, world=2)  # world > 1 needs a unique id
    with pytest.raises(gtc.GTCError) as e:
        gtc.gtc_init(10, 8.0, flags=256)  # no such flag bit
    assert e.value.status == gtc.GTC_EINVAL
    assert gtc.GTC_STEP_SPLIT & (gtc.GTC_CMP_GE | gtc.GTC_EXCHANGE_NCCL) == 0
    with pytest.raises(gtc.GTCError) as e:
        gtc.gtc_init(10, 8.0, world=1, flags=gtc.GTC_LOOPBACK)  # a loopback group has >= 2 ranks
    assert e.value.status == gtc.GTC_EINVAL
    with pytest.raises(gtc.GTCError) as e:
        gtc.gtc_init(10, 8.0, world=2, unique_id=b"\0" * 128, flags=gtc.GTC_LOOPBACK)  # no NCCL id
    assert e.value.status == gtc.GTC_EINVAL
    with pytest.raises(gtc.GTCError) as e:  # the owner-computes decode needs >= 2 ranks
        gtc.gtc_init(10, 8.0, world=1, flags=gtc.GTC_DECODE_SHARDED)
    assert e.value.status == gtc.GTC_EINVAL
    with pytest.raises(gtc.GTCError) as e:  # loopback exchanges p2p only
        gtc.gtc_init(10, 8.0, world=2, flags=gtc.GTC_LOOPBACK | gtc.GTC_EXCHANGE_NCCL)
    assert e.value.status == gtc.GTC_EINVAL
    assert gtc.gtc_strerror(gtc.GTC_ECORRUPT) == "corrupt message"


def test_sm100a_code_in_library():
    import paper_1904_10584_b200 as gtc

    out = subprocess.run(["cuobjdump", "--list-elf", gtc.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1904_10584_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "gtc_oracle" not in txt and "liboracle" not in txt, f
