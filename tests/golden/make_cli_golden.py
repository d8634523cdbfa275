"""Generate tests/golden/cli/ from the REFERENCE command line itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_cli_golden.py

Each case writes an input coefficient file (seeded, numpy PCG64 as in
BASELINE.md §3) and the output file the reference `tftmul` CLI
(pkg/src/tftmul/cli.py, pure-Python path imported from /root/reference)
writes for it; tests/test_cli.py checks that this package's CLI writes the
same bytes.  cases.json lists argv (file names relative to this directory)
and the reference's exit code.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")
sys.path.insert(0, "/root/reference/pkg/src")

from tftmul.cli import main  # noqa: E402  (the reference CLI)


def write_input(name, p, coeffs, root=None):
    lines = [f"p {p}"] + ([f"w {root[0]} {root[1]}"] if root else []) + [str(int(c)) for c in coeffs]
    with open(os.path.join(HERE, name), "w", encoding="ascii") as f:
        f.write("\n".join(lines) + "\n")


def gen(seed, p, n):
    return np.random.default_rng(seed).integers(0, p, n, dtype=np.uint64)


def main_():
    os.makedirs(HERE, exist_ok=True)
    P = 998244353
    write_input("c1000.txt", P, gen(0, P, 1000))                      # config 1 shape, discovered root
    write_input("c777_root.txt", P, gen(5, P, 777), root=(pow(3, 119, P), 23))
    write_input("big_p.txt", 3221225473, gen(6, 3221225473, 1500))    # p > 2^31, discovered ring
    write_input("a300.txt", P, gen(7, P, 300))
    write_input("b201.txt", P, gen(8, P, 201))
    write_input("p17.txt", 17, [5, 0, 11, 3, 9, 16, 2])
    cases = [
        ["tft", "c1000.txt", "c1000.tft.txt"],
        ["itft", "c1000.tft.txt", "c1000.back.txt"],
        ["itft", "c777_root.txt", "c777.itft.txt"],
        ["tft", "big_p.txt", "big_p.tft.txt"],
        ["multiply", "a300.txt", "b201.txt", "prod.txt"],
        ["--modulus", "17", "tft", "p17.txt", "p17_mod.tft.txt"],
        ["--root", "9", "--k", "3", "tft", "p17.txt", "p17_root9.tft.txt"],
        ["--modulus", "3221225473", "tft", "c1000.txt", "c1000_bigp.tft.txt"],
    ]
    cwd = os.getcwd()
    os.chdir(HERE)
    try:
        out = [{"argv": c, "rc": main(c)} for c in cases]
    finally:
        os.chdir(cwd)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("\n".join(f"{c['rc']} {' '.join(c['argv'])}" for c in out))


if __name__ == "__main__":
    main_()
