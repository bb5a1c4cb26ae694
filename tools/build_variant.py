"""Build a debug/experiment variant of libtern.so with extra -D flags into
build/var_<name>/libtern.so (load it with TERN_LIB=...).
python tools/build_variant.py NAME -DFOO=1 [-DBAR=2 ...]"""
import concurrent.futures as cf
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02528_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], tuple(sys.argv[2:])
d = os.path.join(B.ROOT, "build", "var_" + name)
os.makedirs(d, exist_ok=True)
with cf.ThreadPoolExecutor(max_workers=len(B.SOURCES)) as ex:
    objs = list(ex.map(lambda s: B._compile(s, False, d, defs), B.SOURCES))
lib = os.path.join(d, "libtern.so")
r = subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs,
                    "-lcuda"], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(lib)
