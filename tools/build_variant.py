"""Build a variant of libgla.so with extra nvcc defines into variants/ (for A/B runs on one box via GLA_LIB).
python tools/build_variant.py <name> -DFOO=0 ...   ->  variants/libgla_<name>.so"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_06635_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
b.FLAGS_C = b.FLAGS_C + defs
b.FLAGS = b.FLAGS + defs
b.OBJ = "/tmp/gla_obj_" + name
b.LIB = os.path.join(ROOT, "variants", f"libgla_{name}.so")
b.PROBE = f"/tmp/gla_probe_{name}.so"
b.build(force=True)
print(b.LIB)
