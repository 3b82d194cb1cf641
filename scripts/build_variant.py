"""Build a compile-time variant of libhz_b200.so for A/B timing:
  python scripts/build_variant.py NAME -DMACRO=VALUE ...
writes variants/libhz_NAME.so (load it with HZ_LIB_PATH=...)."""
import os, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1607_00968_b200 import build_ext as be
import subprocess

name, defs = sys.argv[1], sys.argv[2:]
root = os.path.join(os.path.dirname(__file__), "..")
obj = os.path.join(root, "variants", "build_" + name)
os.makedirs(obj, exist_ok=True)
out = os.path.join(root, "variants", f"libhz_{name}.so")


def run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)


jobs = [[be.NVCC, *be.FLAGS, *defs, "-c", os.path.join(be.CSRC, s), "-o", os.path.join(obj, s.replace(".cu", ".o"))]
        for s in be.SOURCES]
with ThreadPoolExecutor(8) as ex:
    list(ex.map(run, jobs))
run([be.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out,
     *[os.path.join(obj, s.replace(".cu", ".o")) for s in be.SOURCES], "-cudart", "static"])
print(out)
