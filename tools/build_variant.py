"""Experiment builds of libgtc.so: python tools/build_variant.py OUT.so
[--csrc DIR] [DEFINE ...] -- with -D overrides, or from another source
directory (e.g. a kernel's previous version next to csrc/'s headers, for an
A/B on one box).  Select one at run time with GTC_LIB=OUT.so (not a product
path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10584_b200 import _build  # noqa: E402

if __name__ == "__main__":
    args = sys.argv[2:]
    csrc = None
    if args[:1] == ["--csrc"]:
        csrc, args = os.path.abspath(args[1]), args[2:]
    print(_build.build(force=True, out=os.path.abspath(sys.argv[1]), defines=args, csrc=csrc))
