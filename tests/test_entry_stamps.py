"""Host-side checks of the p2p entry format (csrc/tile_encode.cuh, DESIGN.md
Sec. 7): the helpers are __host__ __device__, so a small host program built
by nvcc exercises exactly the code the kernels use.  No GPU needed."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROG = r"""
#include <cstdio>
#include "tile_encode.cuh"
using namespace gtc;
int main() {
    long bad = 0;
    // stamps: never 0 (0 = cleared slot), and a step's stamp differs from
    // the stamp two steps earlier (same parity), across the 32-bit wrap and
    // the library's epoch sequence (0 is skipped: 0xffffffff -> 1)
    auto next = [](unsigned e) { return e == 0xffffffffu ? 1u : e + 1u; };
    unsigned starts[] = {1u, 524285u, 524287u, 1048573u, 0xffffff00u};
    for (unsigned s0 : starts) {
        unsigned a = s0, b = next(a), c = next(b);
        for (long k = 0; k < 3000000; ++k) {
            if (entry_stamp(a) == 0 || entry_stamp(c) == entry_stamp(a)) ++bad;
            if ((entry_stamp(c) >> 19) != 0) ++bad;   // 19 bits above the 13 of local|neg
            a = b; b = c; c = next(c);
        }
    }
    // entry -> canonical word, every local index and sign, first/last tiles
    long long tiles[] = {0, 1, 5929, (1LL << 31) / kTile - 1};
    for (long long t : tiles)
        for (unsigned l = 0; l < (unsigned)kTile; ++l)
            for (unsigned ng = 0; ng < 2; ++ng) {
                const unsigned st = entry_stamp((unsigned)(l * 7919u + t));
                const unsigned e = make_entry(st, l, ng);
                if ((e >> kStampShift) != st) ++bad;
                const unsigned long long i = (unsigned long long)t * kTile + l;
                if (entry_word(e, t) != (unsigned)((i << 1) | ng)) ++bad;
            }
    // a cleared slot never carries a valid stamp
    for (unsigned e = 1; e < 100000; ++e) if ((0u >> kStampShift) == entry_stamp(e)) ++bad;
    std::printf("bad=%ld\n", bad);
    return bad != 0;
}
"""


def test_entry_stamp_format(tmp_path):
    from paper_1904_10584_b200 import _build

    nvcc = _build.NVCC
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    src = tmp_path / "stamps.cu"
    src.write_text(PROG)
    exe = tmp_path / "stamps"
    cmd = [nvcc, "-std=c++17", "-O1", "-I", os.path.join(ROOT, "paper_1904_10584_b200", "csrc"),
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(_build._nccl_root(), "include"),
           "-o", str(exe), str(src)]
    subprocess.run(cmd, check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "bad=0" in out.stdout, out.stdout + out.stderr
