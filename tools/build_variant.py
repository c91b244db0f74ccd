"""Build an A/B variant of the library with extra -D defines into
tools/_variants/<name>.so (loaded by the *_variants.sh drivers through
MXP_LIB_PATH).  The product build is untouched.

    python tools/build_variant.py k1p_pairs1 -DMXP_K1P_MAX_PAIRS=1
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1204_3052_b200 import build as B  # noqa: E402

name, defines = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(B.ROOT, "tools", "_variants")
obj_dir = os.path.join(out_dir, "_obj_" + name)
os.makedirs(obj_dir, exist_ok=True)


def one(src):
    obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
    cmd = [B.nvcc(), *B.ARCH, *B.FLAGS, *defines, "-c", os.path.join(B.CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return obj


with ThreadPoolExecutor(len(B.SOURCES)) as pool:
    objs = list(pool.map(one, B.SOURCES))
so = os.path.join(out_dir, name + ".so")
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", so, *objs, "-cudart", "static",
                "-Xcompiler", "-fPIC"], check=True)
print(so)
