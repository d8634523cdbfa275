"""The `tftmul`-compatible CLI (paper_1001_5272_b200/cli.py), after the
reference's tests/test_cli.py: file format, exit codes, CSV, selftest.

Argument/format/ring/size failures happen before any device call and run on
CPU; everything that transforms is marked gpu.  The golden cases compare
output files byte-for-byte with the ones the reference CLI wrote
(tests/golden/make_cli_golden.py)."""

import json
import os
import shutil

import pytest

from paper_1001_5272_b200 import RingConfig
from paper_1001_5272_b200.cli import main, parse_coeff_file

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


def coeff_file(path, p, coeffs, root=None):
    lines = [f"p {p}"] + ([f"w {root[0]} {root[1]}"] if root else []) + [str(c) for c in coeffs]
    path.write_text("\n".join(lines) + "\n", encoding="ascii")
    return str(path)


# ---------------------------------------------------------------- CPU
def test_parse_errors_exit_2(tmp_path, capsys):
    dst = str(tmp_path / "out.txt")
    bad = ["q 17\n1\n", "p seventeen\n1\n", "p 17\nw 3\n1\n", "p 17\n", "p 17\n1\ntwo\n", "p 17\n99\n"]
    for text in bad:
        src = tmp_path / "in.txt"
        src.write_text(text, encoding="ascii")
        assert main(["tft", str(src), dst]) == 2, text
    assert main(["tft", str(tmp_path / "missing.txt"), dst]) == 2
    assert capsys.readouterr().err.count("tftmul:") == len(bad) + 1
    assert not os.path.exists(dst)


def test_ring_errors_exit_3(tmp_path):
    dst = str(tmp_path / "out.txt")
    assert main(["tft", coeff_file(tmp_path / "c.txt", 15, [1, 2]), dst]) == 3  # composite
    assert main(["tft", coeff_file(tmp_path / "r.txt", 17, [1, 2], root=(4, 4)), dst]) == 3  # order 4
    a = coeff_file(tmp_path / "a.txt", 17, [1, 2])
    b = coeff_file(tmp_path / "b.txt", 998244353, [1, 2])
    assert main(["multiply", a, b, dst]) == 3


def test_oversize_exits_4(tmp_path):
    dst = str(tmp_path / "out.txt")
    assert main(["tft", coeff_file(tmp_path / "in.txt", 17, [1] * 17), dst]) == 4
    a = coeff_file(tmp_path / "a.txt", 17, [1] * 9)
    assert main(["multiply", a, a, dst]) == 4  # product length 17 > 2^4


def test_root_without_k_exits_2(tmp_path):
    src = coeff_file(tmp_path / "in.txt", 17, [1])
    assert main(["--root", "3", "tft", src, str(tmp_path / "o.txt")]) == 2


def test_missing_subcommand_is_a_usage_error(capsys):
    with pytest.raises(SystemExit) as exc:
        main([])
    assert exc.value.code == 2
    capsys.readouterr()


def test_bench_argument_checks(capsys):
    assert main(["bench", "--nmin", "0", "--nmax", "4"]) == 2
    assert main(["bench", "--nmin", "8", "--nmax", "4"]) == 2
    assert main(["bench", "--nmin", "2", "--nmax", "4", "--trials", "0"]) == 2
    assert main(["bench", "--nmin", "2", "--nmax", str(1 << 24)]) == 4
    capsys.readouterr()


def test_parse_header_forms(tmp_path):
    src = coeff_file(tmp_path / "in.txt", 17, [4, 8, 15], root=(3, 4))
    assert parse_coeff_file(src) == (17, (3, 4), [4, 8, 15])
    src = coeff_file(tmp_path / "in2.txt", 17, [0])
    assert parse_coeff_file(src) == (17, None, [0])


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_transform_file_exact_output_format(tmp_path):
    dst = tmp_path / "out.txt"
    assert main(["tft", coeff_file(tmp_path / "in.txt", 17, [1, 1, 1], root=(3, 4)), str(dst)]) == 0
    assert dst.read_text(encoding="ascii") == "p 17\nw 3 4\n3\n1\n13\n"
    # the same answer when the ring is discovered from p
    assert main(["tft", coeff_file(tmp_path / "in2.txt", 17, [1, 1, 1]), str(dst)]) == 0
    assert dst.read_text(encoding="ascii") == "p 17\nw 3 4\n3\n1\n13\n"


@pytest.mark.gpu
def test_round_trips_reparse_byte_identically(tmp_path):
    src = coeff_file(tmp_path / "in.txt", 17, [4, 8, 15], root=(3, 4))
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    assert main(["tft", src, str(a)]) == 0
    assert main(["itft", str(a), str(b)]) == 0
    assert main(["tft", str(b), str(a)]) == 0
    assert main(["itft", str(a), str(b)]) == 0
    assert b.read_text(encoding="ascii") == "p 17\nw 3 4\n4\n8\n15\n"
    coeffs = [5, 0, 11, 3, 9, 16, 2]
    assert main(["tft", coeff_file(tmp_path / "c.txt", 17, coeffs), str(a)]) == 0
    assert main(["itft", str(a), str(b)]) == 0
    assert parse_coeff_file(str(b)) == (17, (3, 4), coeffs)


@pytest.mark.gpu
def test_single_coefficient_and_product(tmp_path):
    dst = tmp_path / "out.txt"
    assert main(["tft", coeff_file(tmp_path / "in.txt", 17, [13]), str(dst)]) == 0
    assert parse_coeff_file(str(dst))[2] == [13]
    a = coeff_file(tmp_path / "a.txt", 17, [2, 3])
    b = coeff_file(tmp_path / "b.txt", 17, [4, 5, 6])
    assert main(["multiply", a, b, str(dst)]) == 0
    assert parse_coeff_file(str(dst))[2] == [8, 5, 10, 1]


@pytest.mark.gpu
def test_overrides(tmp_path):
    dst = tmp_path / "out.txt"
    src = coeff_file(tmp_path / "in.txt", 998244353, [1, 1, 1], root=(15311432, 23))
    assert main(["--modulus", "17", "tft", src, str(dst)]) == 0  # file root dropped with its modulus
    assert dst.read_text(encoding="ascii") == "p 17\nw 3 4\n3\n1\n13\n"
    src = coeff_file(tmp_path / "in2.txt", 17, [2, 7, 1, 1, 6])
    assert main(["--root", "9", "--k", "3", "tft", src, str(dst)]) == 0
    p, root, got = parse_coeff_file(str(dst))
    assert (p, root) == (17, (9, 3))
    from paper_1001_5272_b200.cli import _naive_dft
    assert got == _naive_dft([2, 7, 1, 1, 6], RingConfig(17, 9, 3))


@pytest.mark.gpu
def test_reference_cli_golden_files(tmp_path):
    """Byte-identical output files vs the reference CLI on the same inputs."""
    with open(os.path.join(GOLD, "cases.json")) as f:
        cases = json.load(f)
    for c in cases:
        for a in c["argv"]:
            if a.endswith(".txt") and os.path.exists(os.path.join(GOLD, a)):
                shutil.copy(os.path.join(GOLD, a), tmp_path / a)
    for c in cases:
        out = c["argv"][-1]
        (tmp_path / out).unlink()
        cwd = os.getcwd()
        os.chdir(tmp_path)
        try:
            assert main(list(c["argv"])) == c["rc"], c["argv"]
        finally:
            os.chdir(cwd)
        with open(os.path.join(GOLD, out), "rb") as f:
            assert (tmp_path / out).read_bytes() == f.read(), c["argv"]


@pytest.mark.gpu
def test_bench_csv(capsys):
    assert main(["bench", "--nmin", "14", "--nmax", "17", "--trials", "1", "--device"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0] == "n,mulcount_tft,mulcount_fft_padded,wall_ns_tft,wall_ns_multiply,dev_ns_tft,dev_ns_fft_padded"
    rows = {int(r.split(",")[0]): [int(v) for v in r.split(",")] for r in lines[1:]}
    assert sorted(rows) == [14, 15, 16, 17]
    for n, (_, mc_tft, mc_fft, wall_t, wall_m, dev_t, dev_f) in rows.items():
        assert mc_tft > 0 and wall_t > 0 and wall_m > 0 and dev_t > 0 and dev_f > 0
        assert mc_tft <= mc_fft + 4 * n
    assert rows[16][1] == rows[16][2]  # power of two: identical tallies
    assert rows[17][1] < rows[17][2]   # just past one: fewer


@pytest.mark.gpu
def test_selftest(capsys, monkeypatch):
    assert main(["selftest"]) == 0
    assert "selftest passed (seed 0)" in capsys.readouterr().out
    monkeypatch.setenv("TFTMUL_SELFTEST_CORRUPT", "1")
    assert main(["selftest", "--seed", "7"]) == 1
    out = capsys.readouterr().out
    assert "selftest FAILED" in out and "--seed 7" in out
