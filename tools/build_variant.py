"""Build a variant of libswr.so with extra nvcc defines into
build_variants/libswr_<tag>.so (kernel-shape experiments; the product
library is built by __graft_entry__.build()).

  python tools/build_variant.py TAG -DNAME=VALUE ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_02564_b200 import _build  # noqa: E402

print(_build.build_variant(sys.argv[1], sys.argv[2:], force=True))
