"""Benchmark driver (contract in the task brief; numbers explained in DESIGN.md).

Default workload = BASELINE config 2, the configuration BASELINE.json's metric
is quoted on that fits one GPU: 4096 independent vectors, lengths uniform in
[2^15+1, 2^16], residues uniform in [0, p), p = 998244353, seed 1 (the pinned
generator of workloads.py).  One step = forward TFT of the whole batch, then
inverse TFT of the whole batch (each direction also timed separately).

  value      2*sum(n) / device time per step, Gcoeff/s (inputs resident in HBM)
  parity     the forward output of the whole batch is checked against the
             sha256 of the REFERENCE's own output (tests/golden/configs.json)
             before anything is timed
  e2e        the same metric through the reference-facing C ABI with HOST
             buffers (tftb_tft_batch_u64 on pinned uint64 words: H2D, convert,
             batch transform, convert, D2H -- once per direction per step)
  e2e_percall  the reference arm's own call pattern: 4096 `_kernels.tft`-shaped
             calls (then 4096 itft) on array('Q') buffers from a
             ThreadPoolExecutor(cores), through backend.kernels()
  roofline   algorithmic bytes (2*passes_min(n)*n*4 per vector
             per direction) / device time of the forward kernel (k_clg_fwd, the
             largest single kernel); roofline_inverse = the split inverse pass;
             against MEASURED_PEAKS.json hbm_gbs
  int_roofline  butterflies (n*ceil_lg(n)/2 per vector, the TFT's own count) /
             device time against the integer-pipe bound of the Shoup
             butterfly (16 per clock per SM) at the measured clock
  config3    BASELINE config 3 at its resolution p = 3221225473 (five lengths
             2^24 .. 2^25+1, seed 2): parity-checked against the reference's
             digests, then fwd/inv timed with L2 flushed between iterations
  cpu_baseline  the reference's own compiled kernels (oracle/_ref, built from
             /root/reference by oracle/Makefile) on a bounded sample of the same
             batch, threaded over vectors on all host cores (they run nogil)

Multi-GPU (torchrun, --gpus N): ONE config-2 batch sharded across the ranks
(shard.shard_ranges: contiguous vector ranges balanced by words); each rank
transforms its shard, then the forward results are gathered to rank 0 over
NCCL (shard.gather_to_root) -- timed separately (gather_ms) -- and rank 0
checks the gathered batch against the reference digest.  value = the whole
batch's coefficients / max-over-ranks step time ("strong" scaling).

--impl reference: the reference CPU path (oracle/_ref) alone, same metric,
rank 0 only.  --config 1|3|4|5 selects the other BASELINE configs for
exploration lines (not the driver's line).
"""

import argparse
import ctypes
import hashlib
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from array import array
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

P = W.P_DEFAULT
TOP = pow(3, 119, P)
KR = 23
SMS = 148
BFLY_PER_CLK_SM = 16  # Shoup butterfly: IMAD.HI (half rate) + 2 IMAD on the FMA pipe


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def golden():
    try:
        with open(os.path.join(ROOT, "tests", "golden", "configs.json")) as f:
            return json.load(f)
    except Exception:
        return None


def sha_words(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def passes_min(n, w=4):
    return 1 if n * w <= 256 * 1024 else 2


def ceil_lg(n):
    return int(n - 1).bit_length()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx.append(float(parts[1]))
                except ValueError:
                    continue
                for nm, val in zip(names, parts[4:8]):
                    if val.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        loaded = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------------ CPU reference
def ref_module():
    from oracle import oracle as O
    mod = O.ref_kernels()
    if mod is None:
        try:
            O.build()
            mod = O.ref_kernels()
        except Exception:
            mod = None
    return mod


def cpu_reference(lens, flat, reps=3, budget_vectors=None, warm=0):
    """Time the reference's compiled kernels (or the oracle port) on a sample
    of the batch, threaded over vectors on all host cores."""
    from oracle import oracle as O
    mod = ref_module()
    kind = "reference" if mod is not None else "port"
    cores = os.cpu_count() or 1
    nvec = budget_vectors or min(len(lens), max(8, 32 * cores))
    offs = np.concatenate(([0], np.cumsum(lens)))
    sample = [(int(offs[i]), int(lens[i])) for i in range(nvec)]
    coeffs = sum(n for _, n in sample)

    def run(direction):
        bufs = [array("Q", flat[o:o + n].tobytes()) for o, n in sample]

        def one(b):
            if mod is not None:
                if direction == "fwd":
                    mod.tft(memoryview(b), 0, len(b), P, TOP, KR)
                else:
                    mod.itft(memoryview(b), 0, len(b), P, TOP, KR, (P + 1) >> 1)
            else:
                a = np.frombuffer(b, dtype=np.uint64)
                r = O.tft(a, P, TOP, KR) if direction == "fwd" else O.itft(a, P, TOP, KR)
                b[:] = array("Q", r.tobytes())
        t0 = time.perf_counter()
        with ThreadPoolExecutor(cores) as ex:
            list(ex.map(one, bufs))
        return time.perf_counter() - t0

    for _ in range(warm):  # untimed warm-up steps
        run("fwd")
        run("inv")
    best_f = min(run("fwd") for _ in range(reps))
    best_i = min(run("inv") for _ in range(reps))
    gcs = 2 * coeffs / (best_f + best_i) / 1e9
    return {"value": gcs, "unit": "Gcoeff/s", "cores": cores, "kind": kind,
            "sample": f"first {nvec} of the 4096 config-2 vectors ({coeffs} coefficients), fwd and inv "
                      f"each best of {reps}, ThreadPoolExecutor({cores}) over vectors "
                      f"({'oracle/_ref = reference _kernels.pyx compiled' if mod else 'oracle C port'})",
            "fwd_gcoeff_s": coeffs / best_f / 1e9, "inv_gcoeff_s": coeffs / best_i / 1e9,
            "sample_ms_per_step": (best_f + best_i) * 1e3}


def reference_arm(args):
    lens, flat = W.c2(1)
    # each step is one bounded sample; best-of over `steps` runs
    res = cpu_reference(lens, flat, reps=max(1, args.steps), warm=args.warmup)
    line = {"metric": "tft_itft_gcoeff_per_s", "value": res["value"], "unit": "Gcoeff/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["sample_ms_per_step"],  # one step = TFT + ITFT of the bounded sample
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (pinned numpy PCG64 generator, seed 1)", "impl": "reference",
            "config": {"workload": "config2: 4096 x n in [2^15+1, 2^16], p=998244353, TFT+ITFT",
                       "sample": res["sample"]},
            "cpu_baseline": res,
            "e2e": {"value": res["value"], "unit": "Gcoeff/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------ GPU legs
def flush_l2(torch, buf):
    buf.add_(1)  # 512 MB read+write: evicts the 126 MB L2


def config3_record(args, T, device, torch, peak, g):
    """Config 3 at p = 3221225473 (BASELINE.md §3 resolution): parity vs the
    reference digest, then fwd/inv device time per length, L2 flushed
    between timed iterations (the vectors are 64-128 MB, near L2 size)."""
    p = W.P_C3
    cfg = T.config_for_modulus(p)
    refs = {r["n"]: r for r in (g or {}).get("config3", []) if r["p"] == p}
    flush = torch.empty(1 << 27, dtype=torch.int32, device="cuda")
    out = []
    reps = max(3, args.steps)
    for n in W.C3_LENGTHS:
        x = W.c3(n, p)
        d = device.to_words(x, cfg)
        device.tft_batch_(d, cfg, n=n)
        got = device.from_words(d, cfg)
        parity = None
        if n in refs:
            parity = sha_words(got) == refs[n]["tft"][0]
            if not parity:
                raise SystemExit(f"config 3 parity failure at n={n}")
        device.tft_batch_(d, cfg, n=n, inverse=True)
        rt = bool(torch.equal(d, device.to_words(x, cfg)))
        ts = {}
        for name, inv in (("fwd", False), ("inv", True)):
            for _ in range(args.warmup):
                device.tft_batch_(d, cfg, n=n, inverse=inv)
            ms = []
            for _ in range(reps):
                flush_l2(torch, flush)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                device.tft_batch_(d, cfg, n=n, inverse=inv)
                b.record()
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
            ts[name] = statistics.median(ms)
        byt = 2 * passes_min(n) * n * 4
        out.append({"n": n, "fwd_ms": ts["fwd"], "inv_ms": ts["inv"],
                    "fwd_gcoeff_s": n / ts["fwd"] / 1e6, "inv_gcoeff_s": n / ts["inv"] / 1e6,
                    "fwd_frac": byt / (ts["fwd"] / 1e3) / 1e9 / peak,
                    "inv_frac": byt / (ts["inv"] / 1e3) / 1e9 / peak,
                    "parity_sha256": parity, "roundtrip_exact": rt})
        del d
    del flush
    torch.cuda.empty_cache()
    return {"p": p, "seed": 2, "l2": "flushed (512 MB write) before every timed iteration; median of "
            f"{reps}", "algorithmic_bytes": "2*2*n*4 per transform (passes_min = 2)", "lengths": out,
            "fwd_frac_min": min(o["fwd_frac"] for o in out), "inv_frac_min": min(o["inv_frac"] for o in out)}


def config4_record(args, T, device, torch, peak, g):
    """Config 4: 256 products 2,500,001 x 1,750,004 (seed 3) in one batched
    multiply (three transforms + fused pointwise product per pair).  Pairs
    0 and 255 are checked against the reference's digests before timing."""
    cfg = T.default_config()
    la, lb, pairs = W.C4_LA, W.C4_LB, W.C4_PAIRS
    r = la + lb - 1
    wd = device.word_dtype(cfg)
    a = torch.empty(pairs * la, dtype=wd, device="cuda")
    b = torch.empty(pairs * lb, dtype=wd, device="cuda")
    for k, pa, pb in W.c4_pairs(range(pairs)):  # one pair at a time: small host footprint
        a[k * la:(k + 1) * la] = device.to_words(pa, cfg)
        b[k * lb:(k + 1) * lb] = device.to_words(pb, cfg)
    x = torch.empty(pairs * r, dtype=wd, device="cuda")
    y = torch.empty(pairs * r, dtype=wd, device="cuda")
    device.multiply_batch(a, b, x, cfg, pairs, la, lb, scratch=y)
    refs = {rec["pair"]: rec["x"] for rec in (g or {}).get("config4", [])}
    parity = {}
    for k in (0, 255):
        if k in refs:
            parity[k] = sha_words(device.from_words(x[k * r:(k + 1) * r], cfg)) == refs[k]
            if not parity[k]:
                raise SystemExit(f"config 4 parity failure at pair {k}")
    for _ in range(args.warmup):
        device.multiply_batch(a, b, x, cfg, pairs, la, lb, scratch=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        device.multiply_batch(a, b, x, cfg, pairs, la, lb, scratch=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    byt = pairs * (4 * (la + lb) + 3 * (2 * passes_min(r) * r * 4) + 3 * r * 4)
    del a, b, x, y
    torch.cuda.empty_cache()
    return {"pairs": pairs, "la": la, "lb": lb, "seed": 3, "ms_per_batch": ms, "products_per_s": pairs / ms * 1e3,
            "roofline_frac": byt / (ms / 1e3) / 1e9 / peak,
            "algorithmic_bytes": "per pair 4(la+lb) + 3*2*2*r*4 + 3*r*4 (SURVEY.md §8(d) 3-transform convention)",
            "parity_sha256_pairs_0_255": parity, "l2": "inputs 4.4 GB > L2; no flush"}


def percall_e2e(T, lens, flat):
    """The reference arm's call pattern through the drop-in: one
    `_kernels.tft` call per vector on an array('Q') buffer, from a thread
    pool (ctypes releases the GIL; each thread leases its own stream)."""
    from paper_1001_5272_b200 import backend
    k = backend.kernels()
    cores = os.cpu_count() or 1
    offs = np.concatenate(([0], np.cumsum(lens)))
    bufs = [array("Q", flat[offs[i]:offs[i + 1]].tobytes()) for i in range(len(lens))]

    def run(inverse):
        def one(b):
            if inverse:
                k.itft(b, 0, len(b), P, TOP, KR, (P + 1) >> 1)
            else:
                k.tft(b, 0, len(b), P, TOP, KR)
        t0 = time.perf_counter()
        with ThreadPoolExecutor(cores) as ex:
            list(ex.map(one, bufs))
        return time.perf_counter() - t0
    run(False)
    run(True)  # warm (contexts, rings, pools)
    tf, ti = run(False), run(True)
    ok = all(np.array_equal(np.frombuffer(b, dtype=np.uint64), flat[offs[i]:offs[i + 1]])
             for i, b in enumerate(bufs))
    total = int(lens.sum())
    return {"value": 2 * total / (tf + ti) / 1e9, "unit": "Gcoeff/s", "calls_per_step": 2 * len(lens),
            "threads": cores, "ms_per_step": (tf + ti) * 1e3, "fwd_ms": tf * 1e3, "inv_ms": ti * 1e3,
            "h2d_bytes_per_step": 2 * 8 * total, "d2h_bytes_per_step": 2 * 8 * total,
            "roundtrip_exact": bool(ok), "timer": "host wall clock (perf_counter) around each pass"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the config-3 sub-record")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args)
        return

    import torch
    import paper_1001_5272_b200 as T
    from paper_1001_5272_b200 import backend, device, shard

    # (BENCH_DIST_BACKEND=gloo: a functional smoke of the multi-rank plumbing
    # on a one-GPU box -- ranks share the device, the gather goes through
    # host memory; never a measurement)
    dist_backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    local = local % max(1, torch.cuda.device_count())
    if args.config != 2:
        explore(args, T, device, backend, torch)
        return
    dist = None
    if world > 1:
        import torch.distributed as dist
        if dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(dist_backend)
    cfg = T.default_config()
    g = golden()
    lens_all, flat_all = W.c2(1)
    # this rank's shard of the ONE batch (contiguous vectors balanced by words)
    s0, s1, lens, offs = shard.local_shard(lens_all, rank, world)
    base = int(np.concatenate(([0], np.cumsum(lens_all)))[s0])
    total = int(lens.sum())
    flat = flat_all[base:base + total]
    d = device.to_words(flat, cfg, device=f"cuda:{local}")
    orig = d.clone()
    stream = torch.cuda.current_stream()
    plan = device.BatchPlan(cfg, lens, offs)

    def fwd():
        plan.execute(d, stream=stream)

    def inv():
        plan.execute(d, inverse=True, stream=stream)

    # ---- parity before timing: the gathered forward output of the whole
    # batch against the reference's digest (rank 0)
    fwd()
    gather_ms = None
    t_g0, t_g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        torch.cuda.synchronize()
        dist.barrier()
        t_g0.record(stream)
        full = shard.gather_to_root(d if dist_backend == "nccl" else d.cpu(), root=0)
        t_g1.record(stream)
        torch.cuda.synchronize()
        gather_ms = t_g0.elapsed_time(t_g1)
    else:
        full = d
    parity = None
    if rank == 0 and g is not None:
        got = device.from_words(full, cfg)
        parity = sha_words(got) == g["config2"]["tft"]
        if not parity:
            raise SystemExit("config 2 parity failure: forward output differs from the reference digest")
    del full
    inv()
    for _ in range(args.warmup):
        fwd()
        inv()
    torch.cuda.synchronize()
    if not torch.equal(d, orig):
        raise SystemExit("round trip failed before timing")

    clocks = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    backend.launch_count(reset=True)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for a, b, c in ev:
        a.record(stream)
        fwd()
        b.record(stream)
        inv()
        c.record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = backend.launch_count()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    fwd_ms = sum(a.elapsed_time(b) for a, b, _ in ev) / args.steps
    inv_ms = sum(b.elapsed_time(c) for _, b, c in ev) / args.steps
    step_ms = t_start.elapsed_time(t_end) / args.steps
    ok = torch.equal(d, orig)

    # ---- end to end through the host-buffer C ABI (pinned uint64 words)
    e2e = None
    if not args.no_e2e:
        host = torch.from_numpy(flat.view(np.int64).copy()).pin_memory()
        hp = host.data_ptr()
        lib = backend.load()
        lp = lens.ctypes.data_as(backend._i64p)
        op = offs.ctypes.data_as(backend._i64p)

        def e2e_step():
            backend.check(lib.tftb_tft_batch_u64(ctypes.c_void_p(hp), op, lp, len(lens), P, TOP, KR, 0))
            backend.check(lib.tftb_tft_batch_u64(ctypes.c_void_p(hp), op, lp, len(lens), P, TOP, KR, 1))
        e2e_step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(torch.cuda.default_stream())
        nrep = max(1, min(args.steps, 3))
        for _ in range(nrep):
            e2e_step()
        t1.record(torch.cuda.default_stream())
        torch.cuda.synchronize()
        e2e_ms = t0.elapsed_time(t1) / nrep
        back = host.numpy().view(np.uint64)
        e2e = {"ms": e2e_ms, "ok": bool(np.array_equal(back, flat))}
        del host

    # ---- reduce over ranks (max time)
    def allmax(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}" if dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}" if dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    step_ms_max = allmax(step_ms)
    fwd_ms_max = allmax(fwd_ms)
    inv_ms_max = allmax(inv_ms)
    coeffs_all = allsum(total)
    ok_all = allsum(0.0 if ok else 1.0) == 0
    alg_bytes_all = float(sum(2 * passes_min(int(n)) * int(n) * 4 for n in lens_all))  # per direction
    bfly_all = float(sum(int(n) * ceil_lg(int(n)) / 2 for n in lens_all))
    e2e_ms_max = allmax(e2e["ms"]) if e2e else None
    e2e_ok = allsum(0.0 if (e2e and e2e["ok"]) else 1.0) == 0 if e2e else None
    gather_ms_max = allmax(gather_ms) if dist else 0.0
    assert coeffs_all == float(lens_all.sum())

    if rank == 0:
        peak, peak_kind = peaks()
        gpus = world
        fwd_ach = alg_bytes_all / (fwd_ms_max / 1e3) / 1e9 / gpus
        inv_ach = alg_bytes_all / (inv_ms_max / 1e3) / 1e9 / gpus
        step_ach = 2 * alg_bytes_all / (step_ms_max / 1e3) / 1e9 / gpus
        clock_ghz = (clk.get("sm_mhz") or 1965.0) / 1e3
        int_peak = BFLY_PER_CLK_SM * SMS * clock_ghz  # Gbfly/s per GPU
        int_fwd = bfly_all / (fwd_ms_max / 1e3) / 1e9 / gpus
        int_inv = bfly_all / (inv_ms_max / 1e3) / 1e9 / gpus
        traffic = {}
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(prof):
            try:
                with open(prof) as f:
                    traffic = json.load(f)
            except Exception:
                traffic = {}
        line = {
            "metric": "tft_itft_gcoeff_per_s",
            "value": 2 * coeffs_all / (step_ms_max / 1e3) / 1e9,
            "unit": "Gcoeff/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": step_ms_max,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic (pinned numpy PCG64 generator, seed 1; workloads.py)",
            "config": {"workload": "config2: one batch of 4096 x n in [2^15+1, 2^16], p=998244353, sharded "
                                   "over the GPUs by words; step = batch TFT then batch ITFT",
                       "global_batch_vectors": int(lens_all.size), "coeffs_total": int(lens_all.sum()),
                       "vectors_rank0": int(lens.size),
                       "l2": "inputs larger than L2 (808 MB vs 126 MB L2 at N=1); no flush",
                       "parallelism": f"dp{world} (one shard per GPU, NCCL gather of results to rank 0)"},
            "parity": {"forward_sha256_vs_reference": parity, "roundtrip_exact": ok_all,
                       "reference": "tests/golden/configs.json config2.tft (reference compiled kernels)"},
            "fwd_gcoeff_s": coeffs_all / (fwd_ms_max / 1e3) / 1e9,
            "inv_gcoeff_s": coeffs_all / (inv_ms_max / 1e3) / 1e9,
            "fwd_ms": fwd_ms_max, "inv_ms": inv_ms_max,
            "kernel_ms": step_ms_max,
            "gather_ms": gather_ms_max,
            "gather_GBps": (4 * coeffs_all * (world - 1) / world / (gather_ms_max / 1e3) / 1e9)
            if world > 1 and gather_ms_max else None,
            "gpu_launches": launches,
            "clocks": clk,
            "roofline": {"bound": "hbm", "kernel": "forward: k_clg_fwd (the largest single kernel)",
                         "achieved": fwd_ach, "peak": peak, "unit": "GB/s", "frac": fwd_ach / peak,
                         "peak_kind": peak_kind, "traffic": traffic.get("forward_bytes"),
                         "note": "algorithmic bytes 2*passes_min(n)*n*4 per vector per direction "
                                 "(BASELINE.md §5) over the pass's CUDA-event time; traffic = ncu "
                                 "dram read+write of the same launches (profiles/traffic.json)"},
            "roofline_inverse": {"bound": "hbm", "kernel": "inverse pass (k_cli_chunks; the last chunk CTA of each vector solves its columns)",
                                 "achieved": inv_ach, "peak": peak, "unit": "GB/s", "frac": inv_ach / peak,
                                 "traffic": traffic.get("inverse_pass_bytes")},
            "roofline_step": {"achieved": step_ach, "frac": step_ach / peak,
                              "traffic": traffic.get("config2_bytes_per_step")},
            "int_roofline": {"bound": "integer pipe", "unit": "Gbutterfly/s",
                             "work": "n*ceil_lg(n)/2 butterflies per vector per direction",
                             "peak": int_peak, "fwd_achieved": int_fwd, "fwd_frac": int_fwd / int_peak,
                             "inv_achieved": int_inv, "inv_frac": int_inv / int_peak,
                             "peak_basis": f"{BFLY_PER_CLK_SM} butterflies/clk/SM x {SMS} SMs x "
                                           f"{clock_ghz:.3f} GHz (measured sm clock)"},
        }
        if e2e:
            line["e2e"] = {"value": 2 * coeffs_all / (e2e_ms_max / 1e3) / 1e9, "unit": "Gcoeff/s",
                           "h2d_bytes_per_step": 2 * 8 * total, "d2h_bytes_per_step": 2 * 8 * total,
                           "ms_per_step": e2e_ms_max, "roundtrip_exact": e2e_ok,
                           "api": "tftb_tft_batch_u64 (pinned host uint64 words), one call per direction"}
        if world == 1:
            if not args.no_e2e:
                line["e2e_percall"] = percall_e2e(T, lens_all, flat_all)
            if not args.no_c3:
                line["config3"] = config3_record(args, T, device, torch, peak, g)
                line["config4"] = config4_record(args, T, device, torch, peak, g)
            if not args.no_cpu:
                line["cpu_baseline"] = cpu_reference(lens_all, flat_all)
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def _time(fn, torch, reps, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def explore(args, T, device, backend, torch):
    """Exploration lines for BASELINE configs 1, 3, 4, 5 (not the driver line),
    on the pinned inputs of workloads.py."""
    peak, _ = peaks()
    out = []
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    if args.config == 1:
        cfg = T.default_config()
        x = W.c1()
        d = device.to_words(x, cfg)
        f = _time(lambda: device.tft_batch_(d, cfg, n=1000), torch, args.steps * 20)
        i = _time(lambda: device.tft_batch_(d, cfg, n=1000, inverse=True), torch, args.steps * 20)
        buf = x.copy()
        t0 = time.perf_counter()
        reps = args.steps * 20
        for _ in range(reps):
            T.tft(buf, cfg)
            T.itft(buf, cfg)
        host_us = (time.perf_counter() - t0) / reps / 2 * 1e6
        out.append({"config": 1, "n": 1000, "fwd_us": f * 1e3, "inv_us": i * 1e3,
                    "host_api_us_per_call": host_us, "roundtrip_exact": bool(np.array_equal(buf, x))})
    elif args.config in (3, 5):
        if args.config == 3:
            cases = [(W.P_C3, n) for n in W.C3_LENGTHS] + [(P, n) for n in W.C3_DEFAULT_LENGTHS]
        else:
            cases = [(W.c5_prime(n, "u32"), n) for n in W.c5_lengths()]
            cases += [(W.P_U64, n) for n in W.c5_lengths()]
        for p, n in cases:
            cfg = T.config_for_modulus(p) if p != P else T.default_config()
            w = 4 if p < (1 << 32) else 8
            batch = W.c5_batch(n, w) if args.config == 5 else 1
            x = W.words(4 if args.config == 5 else 2, p, batch * n)
            d = device.to_words(x, cfg)
            del x
            plan = device.BatchPlan(cfg, np.full(batch, n))
            f = _time(lambda: plan.execute(d), torch, args.steps)
            i = _time(lambda: plan.execute(d, inverse=True), torch, args.steps)
            byt = batch * 2 * passes_min(n, w) * n * w
            out.append({"config": args.config, "p": p, "n": n, "batch": batch,
                        "fwd_ms": f, "inv_ms": i,
                        "fwd_gcoeff_s": batch * n / f / 1e6, "inv_gcoeff_s": batch * n / i / 1e6,
                        "fwd_roofline_frac": byt / (f / 1e3) / 1e9 / peak,
                        "inv_roofline_frac": byt / (i / 1e3) / 1e9 / peak})
            print(json.dumps(out[-1]), flush=True)
            del d, plan
            torch.cuda.empty_cache()
        print(json.dumps({"config": args.config, "clocks": clocks.stop()}))
        return
    elif args.config == 4:
        cfg = T.default_config()
        la, lb, pairs = W.C4_LA, W.C4_LB, W.C4_PAIRS
        r = la + lb - 1
        A, B = W.c4_all()
        a = device.to_words(A, cfg)
        b = device.to_words(B, cfg)
        del A, B
        x = torch.empty(pairs * r, dtype=torch.int32, device="cuda")
        y = torch.empty(pairs * r, dtype=torch.int32, device="cuda")
        t = _time(lambda: device.multiply_batch(a, b, x, cfg, pairs, la, lb, scratch=y), torch, args.steps, warm=1)
        byt = pairs * (4 * (la + lb) + 3 * (2 * 2 * r * 4) + 3 * r * 4)
        out.append({"config": 4, "pairs": pairs, "ms": t, "products_per_s": pairs / t * 1e3,
                    "roofline_frac": byt / (t / 1e3) / 1e9 / peak})
    for o in out:
        print(json.dumps(o))
    print(json.dumps({"config": args.config, "clocks": clocks.stop()}))


if __name__ == "__main__":
    main()
