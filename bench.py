#!/usr/bin/env python
"""Benchmark: mixed-precision Sylvester solves/sec at m=n=4096 (BASELINE.json metric).

A step is one full mp_orth solve (Alg. 3, precision pair binary32/binary64) of
the headline workload "ch": the config-0 recipe at m=n=4096 (A = G_A/sqrt(m)+2I,
B = G_B/sqrt(n)+2I, C ~ N(0,1), seeded synthetic data; the paper's literature
set is not reproduced).  `value` is device-timed with inputs resident in HBM
(L2 flushed between steps); `e2e` goes through the public torch API with pinned
host buffers, H2D of A, B, C and D2H of X inside the timed region.

  python bench.py [--gpus N --steps K --warmup W] [--config ch|c0|c1|c2|c3|c4]
  python bench.py --impl reference ...   # the reference algorithm on the host cores

Multi-GPU (torchrun): one independent replica per rank (a single equation does not
shard), value = total solves / max-over-ranks time, scaling "weak".
"""

from __future__ import annotations

import argparse
import ctypes as ct
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context (see batch.py)
sys.path.insert(0, ROOT)

METRIC = "mixed-precision Sylvester solves/sec at m=n=4096"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="ch", choices=["ch", "c0", "c1", "c2", "c3", "c4"])
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--variant", default="orth", choices=["orth", "inv", "bs"],
                    help="orth/inv: mp_orth / mp_inv (binary32/binary64); bs: fp64 Bartels-Stewart comparator")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-m", type=int, default=512)
    ap.add_argument("--batch", type=int, default=512, help="c4: equations per job (all ranks together)")
    ap.add_argument("--lanes", type=int, default=0, help="c4: concurrent solves per GPU (0 = library default)")
    return ap.parse_args()


def dist_info():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
def cpu_baseline_oracle(m_sample: int, full_m: int, full_n: int, threads: int = 1, reps: int = 1):
    """Time the CPU restatement of the reference (oracle/, a port) on a bounded sample."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle as O  # checker / CPU baseline only
    from paper_2503_03456_b200 import problems as P
    probs = [P.make("c0", m_sample, m_sample, seed=s) for s in range(threads)]
    O.lib()

    def one(p):
        return O.mp_solve(p.A, p.B, p.C, "orth", "binary32")["iterations"]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for _ in range(reps):
            list(ex.map(one, probs))
    dt = time.perf_counter() - t0
    scale = (full_m ** 3 + full_n ** 3) / (2.0 * m_sample ** 3)  # 25(m^3+n^3) Schur flops dominate
    solves = threads * reps
    rate = solves / dt / scale
    return {"value": rate, "unit": "solves/s", "cores": threads, "kind": "port",
            "sample": (f"oracle/ (bit-exact C restatement of the reference mp_orth, binary32/binary64) on "
                       f"{solves} config-0 problems at m=n={m_sample}, {threads} thread(s), {dt:.1f} s; "
                       f"extrapolated to m={full_m}, n={full_n} by the (m^3+n^3) flop law (x{scale:.0f})")}


def run_reference(args):
    rank, local, world = dist_info()
    if rank != 0:
        return
    from paper_2503_03456_b200 import problems as P
    fm, fn = P.FULL_SIZES[args.config]
    fm, fn = args.m or fm, args.n or fn
    threads = min(os.cpu_count() or 1, 64)
    ms = min(args.cpu_sample_m, fm)
    # warm-up: small samples (page in, thread pool)
    for _ in range(args.warmup):
        cpu_baseline_oracle(min(96, ms), fm, fn, threads=threads)
    vals = []
    for _ in range(args.steps):
        vals.append(cpu_baseline_oracle(ms, fm, fn, threads=threads))
    rate = statistics.median(v["value"] for v in vals)
    cb = dict(vals[-1])
    cb["value"] = rate
    line = {
        "metric": METRIC, "value": rate, "unit": "solves/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 / rate if rate > 0 else None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic (seeded, config-0 recipe)",
        "config": {"workload": f"{args.config}: m={fm} n={fn} mp_{args.variant} binary32/binary64",
                   "m": fm, "n": fn},
        "impl": "reference", "cpu_baseline": cb,
        "e2e": {"value": rate, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)



# ---------------------------------------------------------------------------
KCLASSES = ["gemm_dmma_kernel (fp64 DMMA.8x8x4)", "gemm_simt_kernel (fp32/complex FFMA)",
            "apply_z_kernel (window Z application, FFMA)", "chase_kernel (bulge chase, one CTA per chain)",
            "trsyl_step_kernel", "hess_panel kernel", "schur_small/mss (one-CTA Schur)", "aed_kernel"]
KPEAK = {0: "dmma", 1: "ffma", 2: "ffma"}


def ktimer(L, op):
    n = len(KCLASSES)
    cnt, ms, fl = (ct.c_longlong * n)(), (ct.c_double * n)(), (ct.c_double * n)()
    L.sylv_ktimer(op, n, cnt, ms, fl)
    return [(cnt[i], ms[i], fl[i]) for i in range(n)]


KPREFIX = {0: "gemm_dmma", 1: "gemm_simt", 2: "apply_z", 3: "chase", 4: "trsyl", 5: "hess", 6: "schur", 7: "aed"}


def ncu_traffic(cls):
    """Per-launch DRAM bytes of a kernel class from the newest committed `ncu --set full` capture
    (profiles/*ncu_full_capture.json), or (None, None)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_full_capture.json")), key=os.path.getmtime)
    for f in reversed(files):
        try:
            with open(f) as fh:
                cap = json.load(fh)
        except Exception:
            continue
        ls = [l for l in cap.get("launches", []) if l.get("kernel", "").startswith(KPREFIX.get(cls, "?"))]
        if ls:
            return (sum(l["dram_bytes"] for l in ls) / len(ls),
                    f"{os.path.relpath(f, ROOT)}: mean over {len(ls)} captured launches (grids "
                    f"{sorted({l['grid'] for l in ls})})")
    return None, None


def kernel_rooflines(rows, pk, steps):
    """Per kernel class: launches, event-timed ms per step, share of the summed kernel time, achieved
    TFLOP/s from the algorithmic flops declared at each launch.  roofline = the dominant class that
    has an algorithmic flop count."""
    tot = sum(r[1] for r in rows) or 1.0
    out = {}
    for i, (c, ms, fl) in enumerate(rows):
        if c == 0:
            continue
        e = {"launches_per_step": c / steps, "ms_per_step": ms / steps, "share": ms / tot}
        if fl > 0 and ms > 0:
            e["tflops"] = fl / (ms * 1e-3) / 1e12
            pkv = pk.get(KPEAK.get(i))
            if pkv:
                e["frac_of_peak"] = e["tflops"] / pkv
        out[KCLASSES[i]] = e
    best = None
    for i, (c, ms, fl) in enumerate(rows):
        if c and fl > 0 and ms > 0 and (best is None or ms > rows[best][1]):
            best = i
    roof = None
    if best is not None:
        c, ms, fl = rows[best]
        ach = fl / (ms * 1e-3) / 1e12
        peak = pk.get(KPEAK.get(best))
        traffic, tsrc = ncu_traffic(best)
        roof = {"bound": "tensor" if best == 0 else "fp32-simt", "kernel": KCLASSES[best], "achieved": ach,
                "peak": peak, "unit": "TFLOP/s", "frac": ach / peak if peak else None, "traffic": traffic,
                "traffic_source": tsrc,
                "share_of_kernel_time": ms / tot,
                "peak_source": ("measured live by sylv_microbench (DMMA.8x8x4 / FFMA loops); MEASURED_PEAKS.json "
                                "has no fp32/fp64 figure"),
                "algorithmic": (f"{fl / c:.3e} flop per launch (flops declared at each launch from its shapes), "
                                f"{ms / c:.3f} ms average launch, {c / steps:.0f} launches per step; CUDA events "
                                f"on the launching stream around every launch, over a repetition of the K timed "
                                f"steps")}
    return roof, out


def dmma_roofline(L, st, dev, m):
    """Live roofline of the dominant kernel class: the fp64 DMMA GEMM engine (CUDA events on its stream)."""
    import torch
    pk = {}
    for kind, name in ((0, "ffma"), (1, "dfma"), (2, "dmma")):
        v = ct.c_double()
        if L.sylv_microbench(kind, ct.byref(v), ct.c_void_p(st.cuda_stream)) == 0:
            pk[name] = v.value
    g = 4096 if m >= 4096 else max(m, 1024)
    Ga = torch.randn(g, g, dtype=torch.float64, device=dev)
    Gb = torch.randn(g, g, dtype=torch.float64, device=dev)
    Gc = torch.empty(g, g, dtype=torch.float64, device=dev)
    one, zero = ct.c_double(1.0), ct.c_double(0.0)

    def dgemm():
        return L.sylv_gemm(1, b"N", b"N", g, g, g, ct.byref(one), Ga.data_ptr(), g, Gb.data_ptr(), g,
                           ct.byref(zero), Gc.data_ptr(), g, ct.c_void_p(st.cuda_stream))

    for _ in range(3):
        dgemm()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(st)
    nrep = 5
    for _ in range(nrep):
        dgemm()
    a1.record(st)
    a1.synchronize()
    gms = a0.elapsed_time(a1) / nrep
    achieved = 2.0 * g ** 3 / (gms * 1e-3) / 1e12
    peak = pk.get("dmma")
    roof = {"bound": "tensor", "kernel": "gemm_dmma_kernel (fp64 DMMA.8x8x4)", "achieved": achieved,
            "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None, "traffic": None,
            "peak_source": "measured live by sylv_microbench(DMMA) (MEASURED_PEAKS.json has no fp64)",
            "algorithmic": f"2*{g}^3 flop per launch ({g}^3 GEMM), {gms:.2f} ms per launch"}
    return roof, pk


def solve_roofline(pk, variant, kind, m, n, k, cx, t_step, solves_per_step):
    """Paper flop counts (costmodel.flops: low 25a+b fp32, high 6a+(4+3k)b fp64) against the measured peaks."""
    from paper_2503_03456_b200.costmodel import algorithm_name, flops, gemm_phase_flops
    fc = flops(algorithm_name(variant, kind), m, n, k)
    mult = (4.0 if cx else 1.0) * solves_per_step
    low, high = fc.low_flops * mult, fc.high_flops * mult
    p32, p64 = pk.get("ffma"), pk.get("dmma")
    lb = (low / (p32 * 1e12) + high / (p64 * 1e12)) if p32 and p64 else None
    return {"low_flops": low, "high_flops": high, "gflops": (low + high) / t_step / 1e9,
            "frac_of_fp32_fp64_roofline": (lb / t_step) if lb else None,
            "peaks_tflops": pk, "gemm_phase_fp64_flops": gemm_phase_flops(m, n, k) * mult}

# ---------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    rank, local, world = dist_info()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2503_03456_b200 as M
    from paper_2503_03456_b200 import _native, problems as P
    L = _native.lib()
    peaks = measured_peaks()
    fm, fn = P.FULL_SIZES[args.config]
    fm, fn = args.m or fm, args.n or fn
    if args.config == "c4":
        pr = P.make_c4(rank, fm)
    else:
        pr = P.make(args.config, fm, fn, seed=rank)
    m, n = pr.m, pr.n
    cx = pr.is_complex
    dt = torch.complex128 if cx else torch.float64
    A = torch.as_tensor(pr.A, device=dev).to(dt)
    B = torch.as_tensor(pr.B, device=dev).to(dt)
    C = torch.as_tensor(pr.C, device=dev).to(dt)
    X = torch.empty((m, n), dtype=dt, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev)

    def step():
        return M.solve(A, B, C, kind=pr.kind, variant=args.variant, out=X)

    for _ in range(args.warmup):
        _, rep = step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    # ---- device-timed steps (inputs resident in HBM, L2 flushed between steps) ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    reps = []
    launches0 = L.sylv_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            evs[i][0].record(st)
            _, rep = step()
            evs[i][1].record(st)
            reps.append(rep)
        torch.cuda.synchronize(dev)
    launches = (L.sylv_launch_count() - launches0) // max(1, args.steps)
    # per-kernel-class event timing: the same K steps repeated with the library's event
    # timer on (its ~2 event records per launch stay out of `value`)
    ktimer(L, 1)
    for i in range(args.steps):
        flush.fill_(float(i))
        step()
    torch.cuda.synchronize(dev)
    krows = ktimer(L, 2)
    ktimer(L, 0)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = t.item()
        dist.barrier()
    value = world * args.steps / (total_ms / 1e3)
    k = reps[-1].iterations
    # ---- e2e through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        hA = torch.as_tensor(pr.A).to(dt).pin_memory()
        hB = torch.as_tensor(pr.B).to(dt).pin_memory()
        hC = torch.as_tensor(pr.C).to(dt).pin_memory()
        hX = torch.empty((m, n), dtype=dt).pin_memory()
        dA, dB, dC = torch.empty_like(A), torch.empty_like(B), torch.empty_like(C)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        ne = max(1, args.steps)
        for i in range(ne):
            flush.fill_(float(i))
            e0.record(st)
            dA.copy_(hA, non_blocking=True)
            dB.copy_(hB, non_blocking=True)
            dC.copy_(hC, non_blocking=True)
            Xe, _ = M.solve(dA, dB, dC, kind=pr.kind, variant=args.variant)
            hX.copy_(Xe, non_blocking=True)
            e1.record(st)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([tot], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot = t.item()
        esz = hA.element_size()
        e2e = {"value": world * ne / (tot / 1e3), "unit": "solves/s",
               "h2d_bytes_per_step": (m * m + n * n + m * n) * esz, "d2h_bytes_per_step": m * n * esz}
    # ---- roofline: the fp64 DMMA GEMM engine of the contraction phases, timed live ----
    roof = sol_roof = kern = gemm_roof = None
    if rank == 0:
        gemm_roof, pk = dmma_roofline(L, st, dev, m)
        roof, kern = kernel_rooflines(krows, pk, args.steps)
        dm = kern.get(KCLASSES[0])
        if dm and "tflops" in dm:  # the north star's "FP64 tensor peak in its GEMM phases", live in the step
            gemm_roof["in_step"] = {"tflops": dm["tflops"], "frac": dm.get("frac_of_peak"),
                                    "ms_per_step": dm["ms_per_step"]}
        sol_roof = solve_roofline(pk, args.variant, pr.kind, m, n, k, cx, total_ms / args.steps / 1e3, 1)
        sol_roof["phase_ms"] = {"schur": reps[-1].ms_schur, "orth": reps[-1].ms_orth, "setup": reps[-1].ms_setup,
                                "y0": reps[-1].ms_y0, "refine": reps[-1].ms_refine, "recover": reps[-1].ms_recover}
    # ---- CPU baseline (oracle port, rank 0 at N=1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_oracle(min(args.cpu_sample_m, m), m, n, threads=1)
    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": (f"fp64 Bartels-Stewart solves/sec ({args.config}, m={m} n={n})" if args.variant == "bs" else
                       METRIC if args.config == "ch" else f"mixed-precision Sylvester solves/sec ({args.config})"),
            "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32+f64" if not cx else "c64+c128",
            "data": "synthetic (seeded Philox, BASELINE config recipe)",
            "config": {"workload": f"{args.config}: {'complex' if cx else 'real'} {pr.kind} m={m} n={n}, "
                                   f"mp_{args.variant}, precision pair binary32/binary64, one solve per step",
                       "m": m, "n": n, "kind": pr.kind, "variant": args.variant,
                       "l2": "flushed between steps (256 MiB write); working set ~2 GB >> 126 MB L2",
                       "iterations": k, "backward_error": reps[-1].backward_error,
                       "residual": reps[-1].residual,
                       "schur_sweeps": [reps[-1].schur_sweeps_a, reps[-1].schur_sweeps_b],
                       "parallelism": f"replicas x{world}"},
            "roofline": roof, "gemm_phase_roofline": gemm_roof, "kernels": kern, "solve_roofline": sol_roof,
            "cpu_baseline": cpu, "e2e": e2e,
            "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
            "gpu_launches": int(launches),
            "measured_peaks": {"hbm_gbs": peaks.get("hbm_gbs"), "bf16_tflops": peaks.get("bf16_tflops")},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
def run_c4(args):
    """C4: `batch` independent equations (config-0 recipe, m=n=512, entropy seed+i), sharded by equation
    index over the ranks; each rank solves its block with the lane executor (sylv_solve_batched), then one
    gather of X to rank 0 (the only collective).  Total work is fixed as N grows: scaling "strong"."""
    import numpy as np
    import torch
    import torch.distributed as dist
    rank, local, world = dist_info()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2503_03456_b200 as M
    from paper_2503_03456_b200 import _native, problems as P
    from paper_2503_03456_b200.batch import gather_solutions, shard_range
    L = _native.lib()
    peaks = measured_peaks()
    m = args.m or P.FULL_SIZES["c4"][0]
    total = args.batch
    lo, hi = shard_range(total, rank, world)
    cnt = hi - lo
    probs = [P.make_c4(i, m) for i in range(lo, hi)]
    hA = torch.stack([torch.as_tensor(p.A) for p in probs]).pin_memory()
    hB = torch.stack([torch.as_tensor(p.B) for p in probs]).pin_memory()
    hC = torch.stack([torch.as_tensor(p.C) for p in probs]).pin_memory()
    A, B, C = hA.to(dev), hB.to(dev), hC.to(dev)
    X = torch.empty_like(C)
    hX = torch.empty_like(hC).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev)

    def step():
        _, reps = M.solve_batched(A, B, C, out=X, lanes=args.lanes)
        if world > 1:
            gather_solutions(X, total)
        return reps

    for _ in range(args.warmup):
        reps = step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = L.sylv_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            evs[i][0].record(st)
            reps = step()
            evs[i][1].record(st)
        torch.cuda.synchronize(dev)
    launches = (L.sylv_launch_count() - launches0) // max(1, args.steps)
    ktimer(L, 1)  # per-kernel-class event timing over a repetition of the timed steps
    for i in range(args.steps):
        flush.fill_(float(i))
        step()
    torch.cuda.synchronize(dev)
    krows = ktimer(L, 2)
    ktimer(L, 0)
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = t.item()
    value = args.steps * total / (total_ms / 1e3)
    ks = sorted({r.iterations for r in reps})
    st_bad = sum(1 for r in reps if r.status != 0)
    be = max(r.backward_error for r in reps)
    # ---- e2e: pinned host inputs -> device, batched solve, X -> host, gather ----
    e2e = None
    if not args.no_e2e:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for i in range(max(1, args.steps)):
            flush.fill_(float(i))
            e0.record(st)
            A.copy_(hA, non_blocking=True)
            B.copy_(hB, non_blocking=True)
            C.copy_(hC, non_blocking=True)
            M.solve_batched(A, B, C, out=X, lanes=args.lanes)
            hX.copy_(X, non_blocking=True)
            if world > 1:
                gather_solutions(X, total)
            e1.record(st)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([tot], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot = t.item()
        es = hA.element_size()
        e2e = {"value": max(1, args.steps) * total / (tot / 1e3), "unit": "solves/s",
               "h2d_bytes_per_step": cnt * 3 * m * m * es, "d2h_bytes_per_step": cnt * m * m * es}
    roof = sol_roof = cpu = kern = gemm_roof = None
    if rank == 0:
        gemm_roof, pk = dmma_roofline(L, st, dev, m)
        _, kern = kernel_rooflines(krows, pk, args.steps)
        # 64 concurrent lanes: per-launch event intervals include queueing behind the other
        # lanes' kernels, so they cannot give a per-kernel rate; the roofline object is the
        # fp64 DMMA engine on the same (m^3) GEMM shape, timed alone
        roof = dict(gemm_roof)
        roof["note"] = ("C4 runs 64 concurrent solve lanes: the per-class event table ('kernels') measures "
                        "launch-to-completion intervals under contention, not kernel rates")
        sol_roof = solve_roofline(pk, "orth", "general", m, m, max(ks), False, total_ms / args.steps / 1e3,
                                  cnt)
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline_oracle(min(args.cpu_sample_m, m), m, m, threads=1)
    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": f"mixed-precision Sylvester solves/sec (c4: {total} equations, m=n={m})",
            "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic (seeded Philox, entropy seed+index)",
            "config": {"workload": f"c4: {total} x real general m=n={m}, mp_orth binary32/binary64, the whole "
                                   f"batch per step, sharded by equation index + gather of X to rank 0",
                       "m": m, "n": m, "batch": total, "per_rank": cnt, "lanes": args.lanes or 64,
                       "iterations": ks, "failed": st_bad, "max_backward_error": be,
                       "lane_phase_ms_mean": {f: round(sum(getattr(r, "ms_" + f) for r in reps) / len(reps), 2)
                                              for f in ("schur", "orth", "setup", "y0", "refine", "recover",
                                                        "total")},
                       "l2": "flushed between steps (256 MiB write); per-rank working set >> 126 MB L2",
                       "parallelism": f"shard x{world} + gather"},
            "roofline": roof, "gemm_phase_roofline": gemm_roof, "kernels": kern, "solve_roofline": sol_roof,
            "cpu_baseline": cpu, "e2e": e2e,
            "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
            "gpu_launches": int(launches),
            "measured_peaks": {"hbm_gbs": peaks.get("hbm_gbs"), "bf16_tflops": peaks.get("bf16_tflops")},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c4":
        run_c4(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
