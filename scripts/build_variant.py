"""Build a variant of liblodb200.so with extra nvcc -D switches into _variants/<name>.so
(for scripts/ab_lib.sh), leaving the in-tree library as the default build.

    python scripts/build_variant.py NAME [-DFOO=1 ...]
"""
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_14801_b200.build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs(os.path.join(root, "_variants"), exist_ok=True)
B.NVCC_FLAGS = B.NVCC_FLAGS + defs
lib = B.build(force=True)
shutil.copy(lib, os.path.join(root, "_variants", name + ".so"))
B.NVCC_FLAGS = [f for f in B.NVCC_FLAGS if f not in defs]
B.build(force=True)   # restore the default build in-tree
print(name, "built")
