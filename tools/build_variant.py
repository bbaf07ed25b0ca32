"""Tuning builds: python tools/build_variant.py NAME DEF=VAL ... -> paper_1608_04431_b200/libfa_NAME.so
(select with FA_LIB=paper_1608_04431_b200/libfa_NAME.so; never the product library)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04431_b200 import build_native  # noqa: E402

print(build_native.build(variant=sys.argv[1], defines=sys.argv[2:]))
