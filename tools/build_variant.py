"""Experiment builds of libgtc.so with -D overrides (e.g. the warp-specialized
kernel's shape): python tools/build_variant.py OUT.so GTC_WS_GROUPS=3 ...
Select one at run time with GTC_LIB=OUT.so (not a product path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10584_b200 import _build  # noqa: E402

if __name__ == "__main__":
    print(_build.build(force=True, out=os.path.abspath(sys.argv[1]), defines=sys.argv[2:]))
