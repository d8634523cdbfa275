"""Benchmark driver (contract in the task brief; numbers explained in DESIGN.md).

Default workload = BASELINE config 2, the configuration BASELINE.json's metric
is quoted on that fits one GPU: 4096 independent vectors, lengths uniform in
[2^15+1, 2^16], residues uniform in [0, p), p = 998244353, seed 1 (pinned
generator).  One step = forward TFT of the whole batch, then
inverse TFT of the whole batch (each direction also timed separately).

  value      2*sum(n) / device time per step, Gcoeff/s (inputs resident in HBM)
  e2e        same metric through the reference-facing C ABI with HOST buffers
             (tftb_tft_batch_u64 on pinned uint64 words: H2D, convert, batch
             transform, convert, D2H — once per direction per step)
  roofline   algorithmic bytes (2*passes_min(n)*n*4 per vector
             per direction) / device time, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the reference's own compiled kernels (oracle/_ref, built from
             /root/reference by oracle/Makefile) on a bounded sample of the same
             batch, threaded over vectors on all host cores (they run nogil)

Multi-GPU (torchrun): one process per GPU; the global job is N shards of a
config-2-shaped batch (shard r drawn from seed 1+r), one shard per GPU, no
data-path collective (independent vectors); time = max over ranks of the
device time; value = all ranks' coefficients / that time ("weak" scaling).

--impl reference: the reference CPU path (oracle/_ref) alone, same metric,
rank 0 only.  --config 1|3|4|5 selects the other BASELINE configs for
exploration (not the driver's line).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from array import array
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P = 998244353
TOP = pow(3, 119, P)
KR = 23


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def c2_batch(seed):
    rng = np.random.default_rng(seed)
    lens = rng.integers(2 ** 15 + 1, 2 ** 16 + 1, 4096)
    flat = rng.integers(0, P, int(lens.sum()), dtype=np.uint64)
    return lens.astype(np.int64), flat


def passes_min(n, w=4):
    return 1 if n * w <= 256 * 1024 else 2


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


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        lens, flat = c2_batch(1)
        # each step is one bounded sample; best-of over `steps` runs
        res = cpu_reference(lens, flat, reps=max(1, args.steps), warm=args.warmup)
        line = {"metric": "tft_itft_gcoeff_per_s", "value": res["value"], "unit": "Gcoeff/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": res["sample_ms_per_step"],  # one step = TFT + ITFT of the bounded sample
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
                "data": "synthetic (pinned numpy PCG64 generator, seed 1)", "impl": "reference",
                "config": {"workload": "config2: 4096 x n in [2^15+1, 2^16], p=998244353, TFT+ITFT",
                           "sample": res["sample"]},
                "cpu_baseline": res,
                "e2e": {"value": res["value"], "unit": "Gcoeff/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import paper_1001_5272_b200 as T
    from paper_1001_5272_b200 import backend, device

    torch.cuda.set_device(local)
    if args.config != 2:
        explore(args, T, device, backend, torch)
        return
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = T.default_config()
    lens, flat = c2_batch(1 + rank)
    offs = np.concatenate(([0], np.cumsum(lens)[:-1])).astype(np.int64)
    total = int(lens.sum())
    d = device.to_words(flat, cfg, device=f"cuda:{local}")
    orig = d.clone()
    stream = torch.cuda.current_stream()
    plan = device.BatchPlan(cfg, lens, offs)

    def fwd():
        plan.execute(d, stream=stream)

    def inv():
        plan.execute(d, inverse=True, stream=stream)

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
        import ctypes

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
        e2e_ok = bool(np.array_equal(back, flat))
        e2e = {"ms": e2e_ms, "ok": e2e_ok}

    # ---- reduce over ranks (max time)
    def allmax(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    step_ms_max = allmax(step_ms)
    fwd_ms_max = allmax(fwd_ms)
    inv_ms_max = allmax(inv_ms)
    coeffs_all = allsum(total)
    ok_all = allsum(0.0 if ok else 1.0) == 0
    alg_bytes_rank = sum(2 * passes_min(int(n)) * int(n) * 4 for n in lens)  # per direction
    alg_bytes_all = allsum(alg_bytes_rank)
    e2e_ms_max = allmax(e2e["ms"]) if e2e else None

    if rank == 0:
        peak, peak_kind = peaks()
        # dominant kernel: the inverse pass (k_cli_chunks + k_cli_cols, both size classes),
        # its algorithmic bytes over its own event-timed duration, per GPU
        achieved = alg_bytes_all / (inv_ms_max / 1e3) / 1e9 / world
        step_achieved = 2 * alg_bytes_all / (step_ms_max / 1e3) / 1e9 / world
        line = {
            "metric": "tft_itft_gcoeff_per_s",
            "value": 2 * coeffs_all / (step_ms_max / 1e3) / 1e9,
            "unit": "Gcoeff/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": step_ms_max,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic (pinned numpy PCG64 generator, seed 1+rank)",
            "config": {"workload": "config2: 4096 x n in [2^15+1, 2^16] per GPU, p=998244353; "
                                   "step = batch TFT then batch ITFT",
                       "global_batch_vectors": 4096 * world, "coeffs_per_gpu": total,
                       "l2": "inputs larger than L2 (808 MB per GPU vs 126 MB L2); no flush",
                       "parallelism": f"dp{world} (independent shards, no collective)"},
            "fwd_gcoeff_s": coeffs_all / (fwd_ms_max / 1e3) / 1e9,
            "inv_gcoeff_s": coeffs_all / (inv_ms_max / 1e3) / 1e9,
            "fwd_ms": fwd_ms_max, "inv_ms": inv_ms_max,
            "roundtrip_exact": ok_all,
            "gpu_launches": launches,
            "clocks": clk,
            "roofline": {"bound": "hbm", "kernel": "inverse pass (k_cli_chunks + k_cli_cols)", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "peak_kind": peak_kind,
                         "traffic": None,
                         "step_achieved": step_achieved, "step_frac": step_achieved / peak,
                         "note": "algorithmic bytes 2*passes_min(n)*n*4 per vector per direction "
                                 "(BASELINE.md §5) over the pass's CUDA-event time; traffic = ncu "
                                 "dram read+write of the same launches (profiles/traffic.json)"},
        }
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(prof):
            try:
                with open(prof) as f:
                    tj = json.load(f)
                    line["roofline"]["traffic"] = tj.get("inverse_pass_bytes")
                    line["roofline"]["step_traffic"] = tj.get("config2_bytes_per_step")
            except Exception:
                pass
        if e2e:
            line["e2e"] = {"value": 2 * coeffs_all / (e2e_ms_max / 1e3) / 1e9, "unit": "Gcoeff/s",
                           "h2d_bytes_per_step": 2 * 8 * total, "d2h_bytes_per_step": 2 * 8 * total,
                           "ms_per_step": e2e_ms_max, "roundtrip_exact": e2e["ok"]}
        if not args.no_cpu and world == 1:
            line["cpu_baseline"] = cpu_reference(lens, flat)
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
    """Exploration lines for BASELINE configs 1, 3, 4, 5 (not the driver line)."""
    peak, _ = peaks()
    out = []
    if args.config == 1:
        cfg = T.default_config()
        x = np.random.default_rng(0).integers(0, cfg.p, 1000, dtype=np.uint64)
        d = device.to_words(x, cfg)
        f = _time(lambda: device.tft_batch_(d, cfg, n=1000), torch, args.steps * 20)
        i = _time(lambda: device.tft_batch_(d, cfg, n=1000, inverse=True), torch, args.steps * 20)
        out.append({"config": 1, "n": 1000, "fwd_us": f * 1e3, "inv_us": i * 1e3})
    elif args.config in (3, 5):
        c3 = (1 << 24, (1 << 24) + 1, 3 << 23, (1 << 25) - 1, (1 << 25) + 1)
        if args.config == 3:
            # BASELINE.md §3 resolution (p = 3221225473: 2^30 | p-1, canonical u32
            # arithmetic), the same sizes at p = 469762049 = 7 2^26 + 1 (a p < 2^30
            # prime like 998244353, lazy u32 arithmetic), and 998244353's own range
            cases = [(3221225473, n) for n in c3] + [(469762049, n) for n in c3]
            cases += [(998244353, n) for n in (1 << 22, (1 << 22) + 1, 3 << 21, (1 << 23) - 1, 1 << 23)]
        else:
            ns = np.round(np.geomspace(1027, 268435451, 64)).astype(np.int64)
            ns = [int(n) + 1 if n & (n - 1) == 0 else int(n) for n in ns]
            # u32 leg, then the u64 leg (p = 4179340454199820289)
            cases = [(998244353 if n <= (1 << 23) else 3221225473, n) for n in ns]
            cases += [(4179340454199820289, n) for n in ns]
        for p, n in cases:
            cfg = T.config_for_modulus(p) if p != 998244353 else T.default_config()
            sys.stdout.flush()
            batch = max(1, (1 << 28) // n) if args.config == 5 else 1
            w = 4 if p < (1 << 32) else 8
            if batch * n * w > 6e9:
                batch = max(1, int(6e9 // (n * w)))
            if w == 4:
                d = torch.randint(0, 1 << 30, (batch * n,), dtype=torch.int32, device="cuda")
                d.remainder_(p if p < (1 << 31) else (1 << 30))
            else:
                d = torch.randint(0, 1 << 62, (batch * n,), dtype=torch.int64, device="cuda")
                d.remainder_(p)
            try:
                plan = device.BatchPlan(cfg, np.full(batch, n))
            except Exception as e:  # e.g. u64 words beyond the two-pass range (2^26)
                out.append({"config": args.config, "p": p, "n": n, "unsupported": str(e)})
                del d
                continue
            f = _time(lambda: plan.execute(d), torch, args.steps)
            i = _time(lambda: plan.execute(d, inverse=True), torch, args.steps)
            byt = batch * 2 * passes_min(n, w) * n * w
            out.append({"config": args.config, "p": p, "n": n, "batch": batch,
                        "fwd_ms": f, "inv_ms": i,
                        "fwd_gcoeff_s": batch * n / f / 1e6, "inv_gcoeff_s": batch * n / i / 1e6,
                        "fwd_roofline_frac": byt / (f / 1e3) / 1e9 / peak,
                        "inv_roofline_frac": byt / (i / 1e3) / 1e9 / peak})
            del d, plan
            torch.cuda.empty_cache()
    elif args.config == 4:
        cfg = T.default_config()
        la, lb, pairs = 2500001, 1750004, 256
        r = la + lb - 1
        a = torch.randint(0, cfg.p, (pairs * la,), dtype=torch.int32, device="cuda")
        b = torch.randint(0, cfg.p, (pairs * lb,), dtype=torch.int32, device="cuda")
        x = torch.empty(pairs * r, dtype=torch.int32, device="cuda")
        y = torch.empty(pairs * r, dtype=torch.int32, device="cuda")
        t = _time(lambda: device.multiply_batch(a, b, x, cfg, pairs, la, lb, scratch=y), torch, args.steps, warm=1)
        byt = pairs * (4 * (la + lb) + 3 * (2 * 2 * r * 4) + 3 * r * 4)
        out.append({"config": 4, "pairs": pairs, "ms": t, "products_per_s": pairs / t * 1e3,
                    "roofline_frac": byt / (t / 1e3) / 1e9 / peak})
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
