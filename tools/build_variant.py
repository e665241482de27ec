"""Build an A/B variant of the library with extra nvcc defines (probing only).

    python tools/build_variant.py NAME -DFASTRON_X=1 ...  ->  build/variants/lib_NAME.so

Select it at run time with FASTRON_LIB=build/variants/lib_NAME.so (the timing tools print
which library they used)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_06451_b200 import _build  # noqa: E402

name, defines = sys.argv[1], sys.argv[2:]
out = os.path.join(_build.ROOT, "build", "variants")
os.makedirs(out, exist_ok=True)
lib = os.path.join(out, f"lib_{name}.so")
print(_build.build(force=True, extra=defines, lib=lib, objdir=os.path.join(out, f"obj_{name}")))
