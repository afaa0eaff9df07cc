"""Build the library with extra nvcc flags into build/ab/lib<V>.so for a
same-box A/B (tools/ab_lib.sh), without touching the in-tree build.

    python tools/build_variant.py V [-DNAME=VALUE ...]
"""
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06204_b200 import build as Bd  # noqa: E402

if __name__ == "__main__":
    v, extra = sys.argv[1], sys.argv[2:]
    root = Bd.ROOT
    Bd.OBJ = os.path.join(root, "build", "obj_" + v)
    Bd.LIB = os.path.join(root, "build", "ab", "tmp_" + v + ".so")
    Bd.FLAGS = Bd.FLAGS + extra
    os.makedirs(os.path.dirname(Bd.LIB), exist_ok=True)
    out = Bd.build()
    shutil.move(out, os.path.join(root, "build", "ab", "lib" + v + ".so"))
    print("built", os.path.join(root, "build", "ab", "lib" + v + ".so"), extra)
