"""Stage the reference's own test suite against the drop-in.

    python tools/ref_suite.py        # in the build container (needs /root/reference)

Copies the reference package (pure-Python modules + tests; not its Cython
source) into baseline/_ref/refpkg/ -- git-ignored like the rest of
baseline/_ref, so it travels to the GPU box but never enters history -- and
drops integration/_kernels.py in as `tftmul/_kernels.py`.  The GPU test
tests/test_reference_suite.py then runs the reference's pytest suite there:
every `_kernels` call of the reference executes on the B200 through
libtftb200.so.
"""
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg"
DST = os.path.join(ROOT, "baseline", "_ref", "refpkg")

if os.path.exists(DST):
    shutil.rmtree(DST)
os.makedirs(os.path.join(DST, "src"))
shutil.copytree(os.path.join(SRC, "src", "tftmul"), os.path.join(DST, "src", "tftmul"),
                ignore=shutil.ignore_patterns("_kernels*", "__pycache__", "*.so", "*.c"))
shutil.copytree(os.path.join(SRC, "tests"), os.path.join(DST, "tests"),
                ignore=shutil.ignore_patterns("__pycache__"))
shutil.copy(os.path.join(ROOT, "integration", "_kernels.py"), os.path.join(DST, "src", "tftmul", "_kernels.py"))
print("staged", DST)
