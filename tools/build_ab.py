"""Build an A/B variant of the native library with extra -D flags (host tool):
python tools/build_ab.py NAME -DFOO=1 ...  ->  paper_2310_08230_b200/_ab/NAME.so
(load it with DM_LIB_PATH=... for a measurement; never the product path)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2310_08230_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(b.HERE, "_ab")
obj_dir = os.path.join(out_dir, "_obj_" + name)
os.makedirs(obj_dir, exist_ok=True)
env = dict(os.environ)
env.pop("CC", None)
env.pop("CXX", None)
objs = []
for src in b.SOURCES:
    obj = os.path.join(obj_dir, src + ".o")
    subprocess.run([b._nvcc(), *b.ARCH, *b.NVCC_FLAGS, *defs, "-ccbin", "g++", "-c", os.path.join(b.CSRC, src),
                    "-o", obj], check=True, env=env)
    objs.append(obj)
lib = os.path.join(out_dir, name + ".so")
subprocess.run([b._nvcc(), *b.ARCH, "-shared", "-ccbin", "g++", "-o", lib, *objs, "-lcudart"], check=True, env=env)
print(lib)
