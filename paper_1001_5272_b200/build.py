"""Build libtftb200.so in-tree with nvcc for sm_100a (no JIT cache).

    python -m paper_1001_5272_b200.build [--force]
"""

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
UNITS = ["tftb200.cu", "inst_f30.cu", "inst_f32.cu", "inst_f62.cu", "debug.cu", "poly.cu"]
OUT = os.path.join(HERE, "libtftb200.so")
STAMP = OUT + ".stamp"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
OBJ = os.path.join(HERE, "csrc", "_obj")


def _deps(path, seen=None):
    """The unit plus every local header it includes (transitively)."""
    import re
    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    with open(path) as f:
        for m in re.finditer(r'#include\s+"([^"]+)"', f.read()):
            _deps(os.path.normpath(os.path.join(os.path.dirname(path), m.group(1))), seen)
    return seen


def _unit_digest(unit):
    h = hashlib.sha256(" ".join(FLAGS).encode())
    for p in sorted(_deps(os.path.join(HERE, "csrc", unit))):
        with open(p, "rb") as f:
            h.update(os.path.basename(p).encode() + f.read())
    return h.hexdigest()


def _digest():
    h = hashlib.sha256()
    for u in UNITS:
        h.update(_unit_digest(u).encode())
    return h.hexdigest()


def build(force=False, verbose=False):
    """Compile the units whose sources (or local headers) changed, then link."""
    dig = _digest()
    if not force and os.path.exists(OUT) and os.path.exists(STAMP):
        with open(STAMP) as f:
            if f.read().strip() == dig:
                return OUT
    os.makedirs(OBJ, exist_ok=True)
    procs, objs = [], []
    for u in UNITS:
        obj = os.path.join(OBJ, u.replace(".cu", ".o"))
        objs.append(obj)
        ud = _unit_digest(u)
        if not force and os.path.exists(obj) and os.path.exists(obj + ".stamp"):
            with open(obj + ".stamp") as f:
                if f.read().strip() == ud:
                    continue
        cmd = [NVCC, *FLAGS, "-c", "-o", obj, os.path.join(HERE, "csrc", u)]
        procs.append((obj, ud, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    log, failed = "", False
    for obj, ud, pr in procs:
        out, _ = pr.communicate()
        log += f"==== {obj}\n{out}"
        if pr.returncode != 0:
            failed = True
        else:
            with open(obj + ".stamp", "w") as f:
                f.write(ud)
            with open(obj + ".log", "w") as f:
                f.write(out)
    if not failed:
        link = subprocess.run([NVCC, "-shared", "-o", OUT, *objs, "-lcudart"],
                              capture_output=True, text=True)
        log += link.stdout + link.stderr
        failed = link.returncode != 0
    # ptxas.log: every unit's latest register / spill report
    full = ""
    for obj in objs:
        if os.path.exists(obj + ".log"):
            with open(obj + ".log") as f:
                full += f"==== {obj}\n{f.read()}"
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write(full + (log if failed else ""))
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
