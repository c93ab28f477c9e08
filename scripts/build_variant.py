"""Build an experiment variant of libcoserve_cuda.so: the normal objects (build/obj) with the
listed sources recompiled under extra -D flags, linked to paper_2402_18789_b200/variants/<name>.so
(select at run time with CS_LIB_PATH=<that path>).

    python scripts/build_variant.py NAME attn_bwd2.cu[,other.cu] -DFOO -DBAR=2
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_18789_b200 import build as B  # noqa: E402

name, srcs, defs = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
B.build()
vdir = os.path.join(B.PKG, "variants")
odir = os.path.join(B.ROOT, "build", "obj_" + name)
os.makedirs(vdir, exist_ok=True)
os.makedirs(odir, exist_ok=True)
objs = []
for f in sorted(os.listdir(B.OBJ)):
    src = f[:-2]
    if src in srcs:
        o = os.path.join(odir, f)
        cmd = [B.NVCC] + B.ARCH + B.COMMON + defs + ["-c", os.path.join(B.CSRC, src), "-o", o]
        subprocess.run(cmd, check=True)
        objs.append(o)
    else:
        objs.append(os.path.join(B.OBJ, f))
out = os.path.join(vdir, name + ".so")
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", out] + objs +
               ["-lcudart", "-L/usr/lib/x86_64-linux-gnu", "-l:libnccl.so.2"], check=True)
print(out)
