"""Build an experimental variant of libtftb200.so with extra -D flags.

    python tools/build_variant.py NAME [-DKEY=VAL ...]   ->  build/var_NAME/libtftb200.so

Only the F30 units (inst_f30.cu, debug.cu) are recompiled with the flags; the
rest is linked from the main build's objects (run the main build first).
Load it with TFTB_LIB=build/var_NAME/libtftb200.so (backend.py).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1001_5272_b200.build import FLAGS, HERE, NVCC, OBJ, UNITS  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "build", f"var_{name}")
os.makedirs(out, exist_ok=True)
redo = ["inst_f30.cu", "debug.cu"]
procs = []
for u in redo:
    o = os.path.join(out, u.replace(".cu", ".o"))
    procs.append(subprocess.Popen([NVCC, *FLAGS, *defs, "-c", "-o", o, os.path.join(HERE, "csrc", u)],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
logs = [p.communicate()[0] for p in procs]
if any(p.returncode for p in procs):
    sys.stderr.write("\n".join(logs))
    sys.exit(1)
objs = [os.path.join(out, u.replace(".cu", ".o")) if u in redo else os.path.join(OBJ, u.replace(".cu", ".o"))
        for u in UNITS]
subprocess.run([NVCC, "-shared", "-o", os.path.join(out, "libtftb200.so"), *objs, "-lcudart"], check=True)
with open(os.path.join(out, "ptxas.log"), "w") as f:
    f.write("\n".join(logs))
print(os.path.join(out, "libtftb200.so"))
