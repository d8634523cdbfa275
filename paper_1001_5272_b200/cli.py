"""`tftmul`-compatible command line on the B200 path.

Same subcommands, coefficient-file format, output bytes and exit codes as
the reference front end (pkg/src/tftmul/cli.py:1-19, 272-316), so scripts
written against `tftmul` keep working; every transform and product runs
through this package's GPU path (tft / itft / multiply -> libtftb200).

File format (cli.py:3-12 of the reference): decimal, one item per line,

    p <modulus>
    w <root> <k>        optional; root of order exactly 2^k
    <coefficient>       one per line, in [0, p)

Written files always carry both header lines, so they re-parse
byte-identically.  Exit codes: 0 ok, 2 malformed input, 3 bad modulus or
root, 4 length beyond 2^K (cli.py:42-44).

    python -m paper_1001_5272_b200 tft in.txt out.txt
    python -m paper_1001_5272_b200 bench --nmin 2 --nmax 128 [--device]
    python -m paper_1001_5272_b200 selftest [--seed S]
"""

import argparse
import os
import random
import sys
import time

from . import backend
from .modring import (
    RingConfig,
    RingConfigError,
    UnsupportedSizeError,
    ceil_lg,
    config_for_modulus,
    default_config,
    make_buffer,
    zeros,
)
from .polymul import multiply
from .transforms import fft_pow2, itft, tft

EXIT_OK, EXIT_PARSE, EXIT_RING, EXIT_SIZE = 0, 2, 3, 4
CSV_HEADER = "n,mulcount_tft,mulcount_fft_padded,wall_ns_tft,wall_ns_multiply"
DEVICE_COLUMNS = ",dev_ns_tft,dev_ns_fft_padded"
# the default ring's transform of (1, 2, 3, 4) (reference cli.py:42, 232-235)
DEFAULT_RING_ANSWER = (10, 998244351, 173167434, 825076915)


class CliError(Exception):
    """A user-facing failure with the process exit code it maps to."""

    def __init__(self, code, message):
        super().__init__(message)
        self.code = code


# ------------------------------------------------------------- file I/O
def _int_field(text, path, what):
    try:
        return int(text)
    except ValueError:
        raise CliError(EXIT_PARSE, f"{path}: bad {what} {text!r}") from None


def parse_coeff_file(path):
    """(p, (root, k) or None, coefficients) of a coefficient file.  Only the
    shape is checked here; ranges are checked once the ring is known."""
    try:
        with open(path, "r", encoding="ascii") as fh:
            body = [t.strip() for t in fh.read().splitlines()]
    except OSError as e:
        raise CliError(EXIT_PARSE, f"{path}: {e.strerror or e}") from e
    body = [t for t in body if t]
    if not body or not body[0].startswith("p "):
        raise CliError(EXIT_PARSE, f"{path}: first line must be 'p <modulus>'")
    p = _int_field(body[0][2:], path, "modulus line")
    root, first = None, 1
    if len(body) > 1 and body[1].startswith("w "):
        fields = body[1].split()
        if len(fields) != 3:
            raise CliError(EXIT_PARSE, f"{path}: bad root line {body[1]!r}")
        root = (_int_field(fields[1], path, "root line"), _int_field(fields[2], path, "root line"))
        first = 2
    coeffs = [_int_field(t, path, "coefficient") for t in body[first:]]
    if not coeffs:
        raise CliError(EXIT_PARSE, f"{path}: no coefficients")
    return p, root, coeffs


def write_coeff_file(path, cfg, coeffs):
    lines = [f"p {cfg.p}", f"w {cfg.omegaK} {cfg.K}"] + [str(c) for c in coeffs]
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(lines) + "\n")


def build_config(file_p, file_root, args):
    """The ring after --modulus / --root / --k overrides.  A root read from a
    file belongs to the file's modulus and is dropped when --modulus
    changes it (reference test_cli.py:113-119)."""
    if (args.root is None) != (args.k is None):
        raise CliError(EXIT_PARSE, "--root and --k must be given together")
    p = file_p if args.modulus is None else args.modulus
    if args.root is not None:
        root = (args.root, args.k)
    else:
        root = file_root if p == file_p else None
    try:
        return config_for_modulus(p) if root is None else RingConfig(p, root[0], root[1])
    except RingConfigError as e:
        raise CliError(EXIT_RING, str(e)) from e


def _read_operand(path, args):
    p, root, coeffs = parse_coeff_file(path)
    cfg = build_config(p, root, args)
    bad = next((c for c in coeffs if not 0 <= c < cfg.p), None)
    if bad is not None:
        raise CliError(EXIT_PARSE, f"{path}: coefficient {bad} outside [0, {cfg.p})")
    return cfg, coeffs


def _same_ring(a, b):
    return (a.p, a.omegaK, a.K) == (b.p, b.omegaK, b.K)


# ----------------------------------------------------------- subcommands
def run_transform(args):
    cfg, coeffs = _read_operand(args.infile, args)
    buf = make_buffer(coeffs, cfg)
    try:
        (itft if args.command == "itft" else tft)(buf, cfg)
    except UnsupportedSizeError as e:
        raise CliError(EXIT_SIZE, str(e)) from e
    write_coeff_file(args.outfile, cfg, buf)
    return EXIT_OK


def run_multiply(args):
    cfg, a = _read_operand(args.afile, args)
    cfg_b, b = _read_operand(args.bfile, args)
    if not _same_ring(cfg, cfg_b):
        raise CliError(EXIT_RING, "input files use different rings")
    out = zeros(len(a) + len(b) - 1, cfg)
    try:
        multiply(make_buffer(a, cfg), make_buffer(b, cfg), out, cfg)
    except UnsupportedSizeError as e:
        raise CliError(EXIT_SIZE, str(e)) from e
    write_coeff_file(args.outfile, cfg, out)
    return EXIT_OK


def _best_ns(trials, fn):
    best = None
    for _ in range(trials):
        t0 = time.perf_counter_ns()
        fn()
        dt = time.perf_counter_ns() - t0
        best = dt if best is None else min(best, dt)
    return best


def _device_ns(n, cfg, trials):
    """Best-of-`trials` CUDA-event time of the in-HBM transform of one
    n-word vector (words already resident: kernels only)."""
    import torch

    from . import device

    words = device.to_words(list(range(n)), cfg)
    best = None
    for _ in range(trials + 1):  # first call warms the plan caches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        device.tft_batch_(words, cfg, n=n)
        e1.record()
        e1.synchronize()
        ns = int(e0.elapsed_time(e1) * 1e6)
        best = ns if best is None else min(best, ns)
    return best


def run_bench(args):
    """CSV per length: the reference's op tallies of the TFT and of the
    padded power-of-two transform, and GPU wall times through the public API
    (host buffers in and out).  --device adds kernel-only times of the TFT
    and of the padded transform, the smoothness the TFT is for."""
    if not 1 <= args.nmin <= args.nmax:
        raise CliError(EXIT_PARSE, "need 1 <= nmin <= nmax")
    if args.trials < 1:
        raise CliError(EXIT_PARSE, "need at least one trial")
    tally_cfg, cfg = default_config(instrument=True), default_config()
    if args.nmax > 1 << cfg.K:
        raise CliError(EXIT_SIZE, f"nmax {args.nmax} exceeds 2^{cfg.K}")
    rng = random.Random(0)
    emit = sys.stdout.write
    emit(CSV_HEADER + (DEVICE_COLUMNS if args.device else "") + "\n")
    for n in range(args.nmin, args.nmax + 1):
        data = [rng.randrange(cfg.p) for _ in range(n)]
        counts = []
        for buf, fn in ((make_buffer(data, tally_cfg), tft), (zeros(1 << ceil_lg(n), tally_cfg), fft_pow2)):
            tally_cfg.counters.reset()
            fn(buf, tally_cfg)
            counts.append(tally_cfg.counters.mults)
        t_tft = _best_ns(args.trials, lambda: tft(make_buffer(data, cfg), cfg))
        half = (n + 1) // 2  # operands sized so the product has n coefficients
        a = make_buffer([rng.randrange(cfg.p) for _ in range(half)], cfg)
        b = make_buffer([rng.randrange(cfg.p) for _ in range(n + 1 - half)], cfg)
        prod = zeros(n, cfg)
        t_mul = _best_ns(args.trials, lambda: multiply(a, b, prod, cfg))
        row = [n, counts[0], counts[1], t_tft, t_mul]
        if args.device:
            row += [_device_ns(n, cfg, args.trials), _device_ns(1 << ceil_lg(n), cfg, args.trials)]
        emit(",".join(str(v) for v in row) + "\n")
    return EXIT_OK


def _naive_dft(coeffs, cfg):
    """Quadratic evaluation at omega_s, s < n: the self test's independent
    checker (the reference's oracle.naive_dft, oracle.py:46-63), CPU-side
    and used for nothing but comparison."""
    from .modring import omega
    p = cfg.p
    out = []
    for s in range(len(coeffs)):
        w, acc = omega(s, cfg), 0
        for c in reversed(coeffs):
            acc = (acc * w + c) % p
        out.append(acc)
    return out


def _schoolbook(a, b, p):
    """Quadratic product (reference oracle.schoolbook_mul, oracle.py:66-76)."""
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] = (out[i + j] + x * y) % p
    return out


def _selftest_checks(cfg, rng):
    """Yield (description, ok) for each check, in the reference's order
    (cli.py:205-269); the footprint audit replaces audited_call."""
    try:
        RingConfig(cfg.p, cfg.omegaK, cfg.K)
        yield "ring validation", True
    except RingConfigError as e:
        yield f"ring validation ({e})", False
        return
    small = RingConfig(17, 3, 4)
    buf = make_buffer([1, 1, 1], small)
    tft(buf, small)
    yield "fixed transform answer over p=17", list(buf) == [3, 1, 13]
    out = zeros(4, small)
    multiply(make_buffer([2, 3], small), make_buffer([4, 5, 6], small), out, small)
    yield "fixed product answer over p=17", list(out) == [8, 5, 10, 1]
    buf = make_buffer([1, 2, 3, 4], cfg)
    tft(buf, cfg)
    yield "fixed transform answer over the default modulus", tuple(buf) == DEFAULT_RING_ANSWER
    for n in range(1, 97):
        data = [rng.randrange(cfg.p) for _ in range(n)]
        buf = make_buffer(data, cfg)
        tft(buf, cfg)
        if n <= 48:
            yield f"oracle mismatch at n={n}", list(buf) == _naive_dft(data, cfg)
        itft(buf, cfg)
        yield f"round trip at n={n}", list(buf) == data
    for _ in range(30):
        la, lb = rng.randrange(1, 25), rng.randrange(1, 25)
        a = [rng.randrange(cfg.p) for _ in range(la)]
        b = [rng.randrange(cfg.p) for _ in range(lb)]
        out = zeros(la + lb - 1, cfg)
        multiply(make_buffer(a, cfg), make_buffer(b, cfg), out, cfg)
        yield f"product mismatch at {la}x{lb}", list(out) == _schoolbook(a, b, cfg.p)
    # footprint audit: the transform needs no device memory beyond its n words
    aux = {}
    for n in (16, 512):
        buf = make_buffer([rng.randrange(cfg.p) for _ in range(n)], cfg)
        backend.aux_bytes(reset=True)
        tft(buf, cfg)
        aux[n] = backend.aux_bytes()
    yield "transform allocated a buffer", aux[16] == 0 and aux[512] == 0


def run_selftest(args):
    cfg = default_config(instrument=True)
    if os.environ.get("TFTMUL_SELFTEST_CORRUPT"):
        cfg.omegaK += 1  # the reference's sabotage hook (cli.py:209-211)
    for what, ok in _selftest_checks(cfg, random.Random(args.seed)):
        if not ok:
            print(f"selftest FAILED: {what}; reproduce with --seed {args.seed}")
            return 1
    print(f"selftest passed (seed {args.seed})")
    return EXIT_OK


# ------------------------------------------------------------------ main
def _parser():
    ap = argparse.ArgumentParser(
        prog="tftmul",
        description="Arbitrary-length in-place transforms and products over a prime field (B200).")
    ap.add_argument("--modulus", type=int, help="override the file modulus")
    ap.add_argument("--root", type=int, help="override the file root (needs --k)")
    ap.add_argument("--k", type=int, help="power-of-two order of --root")
    sub = ap.add_subparsers(dest="command", required=True)
    for name, what in (("tft", "forward"), ("itft", "inverse")):
        sp = sub.add_parser(name, help=f"{what} transform of a coefficient file")
        sp.add_argument("infile")
        sp.add_argument("outfile")
    sp = sub.add_parser("multiply", help="polynomial product of two files")
    for f in ("afile", "bfile", "outfile"):
        sp.add_argument(f)
    sp = sub.add_parser("bench", help="CSV of counts and wall times per length")
    sp.add_argument("--nmin", type=int, default=2)
    sp.add_argument("--nmax", type=int, default=128)
    sp.add_argument("--trials", type=int, default=3)
    sp.add_argument("--device", action="store_true", help="add kernel-only GPU times (TFT, padded pow2)")
    sp = sub.add_parser("selftest", help="run the reduced validation suite")
    sp.add_argument("--seed", type=int, default=0)
    return ap


COMMANDS = {"tft": run_transform, "itft": run_transform, "multiply": run_multiply,
            "bench": run_bench, "selftest": run_selftest}


def main(argv=None):
    args = _parser().parse_args(argv)
    try:
        return COMMANDS[args.command](args)
    except CliError as e:
        print(f"tftmul: {e}", file=sys.stderr)
        return e.code


def entry():
    sys.exit(main())


if __name__ == "__main__":
    entry()
