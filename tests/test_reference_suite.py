"""The reference's OWN test suite, run with integration/_kernels.py as its
`tftmul._kernels` (every compiled-path call executes on the B200 through
libtftb200.so).  Staged by tools/ref_suite.py into baseline/_ref/refpkg
(git-ignored, travels with the working tree); skipped when absent."""

import os
import re
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "baseline", "_ref", "refpkg")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not os.path.isdir(PKG), reason="run tools/ref_suite.py to stage the reference suite")]


def test_reference_suite_through_the_drop_in():
    env = dict(os.environ, PYTHONPATH=os.path.join(PKG, "src"),
               TFTB_LIB=os.path.join(ROOT, "paper_1001_5272_b200", "libtftb200.so"))
    env.pop("TFTMUL_BACKEND", None)
    probe = subprocess.run([sys.executable, "-c", "from tftmul import backend, _kernels; "
                            "print(backend.backend_name(), _kernels.__file__)"],
                           env=env, capture_output=True, text=True, cwd=PKG)
    assert probe.returncode == 0, probe.stderr
    name, path = probe.stdout.split()
    assert name == "compiled" and path.endswith("_kernels.py")
    r = subprocess.run([sys.executable, "-m", "pytest", "tests", "-q", "-p", "no:cacheprovider"],
                       env=env, capture_output=True, text=True, cwd=PKG, timeout=1800)
    tail = r.stdout[-3000:]
    assert r.returncode == 0, tail + r.stderr[-2000:]
    m = re.search(r"(\d+) passed", tail)
    assert m and int(m.group(1)) >= 90, tail
    assert "failed" not in tail.splitlines()[-1], tail
