"""Build a variant of libmgb.so with extra nvcc flags into its own path (A/B runs on the GPU box):

python tools/build_variant.py OUT.so -DMGB_MLA_SACC=2 ...   then   MGB_LIB=OUT.so python ...
"""
import os
import subprocess
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200 import build as B  # noqa: E402

out, extra = Path(sys.argv[1]), sys.argv[2:]
tmp = Path(tempfile.mkdtemp())
objs = []
for src in B._sources():
    obj = tmp / (src.name.replace(".", "_") + ".o")
    if src.suffix == ".cpp":
        cmd = [B.CXX, *B.CXX_FLAGS, "-c", str(src), "-o", str(obj)]
    else:
        flags = list(B.NVCC_FLAGS)
        i = flags.index("-v")
        del flags[i - 1:i + 1]  # drop "-Xptxas -v"
        cmd = [B.NVCC, *B.ARCH_FLAGS, *flags, *extra, "-c", str(src), "-o", str(obj)]
    pr = subprocess.run(cmd, capture_output=True, text=True)
    if pr.returncode:
        sys.exit(f"{src.name}: {pr.stderr[-2000:]}")
    objs.append(str(obj))
subprocess.run([B.NVCC, *B.ARCH_FLAGS, "-shared", "-o", str(out), *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"],
               check=True)
print(f"built {out} with {' '.join(extra)}")
