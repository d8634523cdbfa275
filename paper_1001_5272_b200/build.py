"""Build libtftb200.so in-tree with nvcc for sm_100a (no JIT cache).

    python -m paper_1001_5272_b200.build [--force]
"""

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
UNITS = ["tftb200.cu", "inst_f30.cu", "inst_f32.cu", "inst_f62.cu", "debug.cu"]
OUT = os.path.join(HERE, "libtftb200.so")
STAMP = OUT + ".stamp"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
OBJ = os.path.join(HERE, "csrc", "_obj")


def _digest():
    h = hashlib.sha256(" ".join(FLAGS).encode())
    for d in (os.path.join(HERE, "csrc"), os.path.join(ROOT, "include")):
        for name in sorted(os.listdir(d)):
            if os.path.isdir(os.path.join(d, name)):
                continue
            with open(os.path.join(d, name), "rb") as f:
                h.update(name.encode() + f.read())
    return h.hexdigest()


def build(force=False, verbose=False):
    dig = _digest()
    if not force and os.path.exists(OUT) and os.path.exists(STAMP):
        with open(STAMP) as f:
            if f.read().strip() == dig:
                return OUT
    os.makedirs(OBJ, exist_ok=True)
    procs = []
    for u in UNITS:
        obj = os.path.join(OBJ, u.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, "-c", "-o", obj, os.path.join(HERE, "csrc", u)]
        procs.append((obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    log, failed = "", False
    for obj, pr in procs:
        out, _ = pr.communicate()
        log += f"==== {obj}\n{out}"
        failed |= pr.returncode != 0
    if not failed:
        link = subprocess.run([NVCC, "-shared", "-o", OUT, *[o for o, _ in procs], "-lcudart"],
                              capture_output=True, text=True)
        log += link.stdout + link.stderr
        failed = link.returncode != 0
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write(log)
    if failed:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed building libtftb200.so")
    if verbose:
        sys.stdout.write(log)
    with open(STAMP, "w") as f:
        f.write(dig)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
