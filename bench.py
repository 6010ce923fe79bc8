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
    ap.add_argument("--cpu-sample-m", type=int, default=1024,
                    help="size of the oracle sample behind cpu_baseline / --impl reference (extrapolated)")
    ap.add_argument("--correction", type=int, default=64, choices=[64, 32],
                    help="precision of the correction solve in Alg. 1 (64 = the reference; 32 = the fast mode)")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 sharded-batch sub-measurement")
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
def cpu_baseline_oracle(m_sample: int, full_m: int, full_n: int, threads: int = 0, config: str = "c0"):
    """Time the CPU restatement of the reference (oracle/, a port of the reference's algorithm, bit-exact in
    binary32) on ONE bounded sample solve at m=n=m_sample, using `threads` host threads (OpenMP across the
    independent entries of each step; 0 = all cores), and extrapolate to (full_m, full_n) by the
    alpha = m^3 + n^3 law of the Schur-dominated flop count.  Returns the cpu_baseline dict."""
    from oracle import oracle as O  # checker / CPU baseline only
    from paper_2503_03456_b200 import problems as P
    threads = threads or (os.cpu_count() or 1)
    used = O.lib().oracle_set_threads(threads)
    cfg = config if config in ("c0", "c1", "c3", "ch") else "c0"
    p = P.make(cfg, m_sample, m_sample if cfg != "c1" else None, seed=0)
    t0 = time.perf_counter()
    rep = O.mp_solve(p.A, p.B, p.C, "orth", "binary32", p.kind)
    dt = time.perf_counter() - t0
    scale = (full_m ** 3 + full_n ** 3) / (p.m ** 3 + p.n ** 3)
    rate = 1.0 / dt / scale
    return {"value": rate, "unit": "solves/s", "cores": used, "kind": "port",
            "sample": (f"oracle/ (C restatement of the reference mp_orth, bit-exact in binary32) on one {cfg}-recipe "
                       f"problem at m={p.m} n={p.n} (k={rep['iterations']}), {used} OpenMP thread(s): {dt:.2f} s; "
                       f"EXTRAPOLATED to m={full_m}, n={full_n} by the alpha = m^3+n^3 law (x{scale:.0f})"),
            "extrapolated": {"from_m": p.m, "from_n": p.n, "to_m": full_m, "to_n": full_n, "factor": scale,
                             "law": "alpha = m^3 + n^3", "sample_seconds": dt},
            "sample_seconds": dt}


def cpu_baseline_python(config: str, m: int, n: int):
    """The UNMODIFIED reference (baseline/_ref, pure Python + numpy) timed on its own public API,
    mpsylv.mp_orth, at the full size of a config it finishes in minutes (C0: m=n=128).  None if the
    reference install is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "mpsylv")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import mpsylv
    from paper_2503_03456_b200 import problems as P
    p = P.make(config, m, n, seed=0)
    prob = mpsylv.SylvesterProblem(p.A, p.B, p.C, kind=p.kind)
    cfg = mpsylv.RefinementConfig(mpsylv.BINARY32, mpsylv.BINARY64)
    t0 = time.perf_counter()
    rep = mpsylv.mp_orth(prob, cfg)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": "solves/s", "cores": 1, "kind": "reference",
            "sample": (f"baseline/_ref mpsylv.mp_orth (the unmodified reference, interpreted Python + numpy) on the "
                       f"{config} problem at full size m={m} n={n}: {dt:.1f} s, k={rep.iterations}, residual "
                       f"{rep.residual:.2e}"),
            "sample_seconds": dt}


def run_reference(args):
    """The reference arm.  C0: the unmodified Python reference (baseline/_ref) at full size, one solve per
    step.  Other configs: the oracle port of the reference algorithm with every host thread, one bounded
    sample solve per step, the metric extrapolated to the config's size (the Python reference takes hours to
    days there) and labelled so; ms_per_step is the measured time of the steps actually run."""
    rank, local, world = dist_info()
    if rank != 0:
        return
    from paper_2503_03456_b200 import problems as P
    fm, fn = P.FULL_SIZES[args.config]
    fm, fn = args.m or fm, args.n or fn
    vals = []
    use_python = args.config == "c0" and os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "mpsylv"))
    for i in range(args.warmup + args.steps):
        if use_python:
            v = cpu_baseline_python("c0", fm, fn)
        else:
            v = cpu_baseline_oracle(min(args.cpu_sample_m, fm) if i >= args.warmup else min(256, fm), fm, fn,
                                    config=args.config)
        if i >= args.warmup:
            vals.append(v)
    rate = statistics.median(v["value"] for v in vals)
    step_s = [v["sample_seconds"] for v in vals]
    cb = dict(vals[-1])
    cb["value"] = rate
    line = {
        "metric": METRIC if args.config == "ch" else f"mixed-precision Sylvester solves/sec ({args.config})",
        "value": rate, "unit": "solves/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(step_s), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic (seeded, config recipe)",
        "config": {"workload": f"{args.config}: m={fm} n={fn} mp_orth binary32/binary64", "m": fm, "n": fn},
        "impl": "reference", "cpu_baseline": cb,
        "extrapolated": cb.get("extrapolated") is not None,
        "e2e": {"value": rate, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if cb.get("extrapolated"):
        line["extrapolation"] = dict(cb["extrapolated"], note=(
            "ms_per_step is the measured time of each sample solve actually run; value is that rate scaled to the "
            "config's size by the flop law"))
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
    """Per-launch DRAM bytes (read + write) of a kernel class from the newest committed `ncu --set
    full` summary (profiles/r*_ncu_full_kernels.json, or the older *ncu_full_capture.json), or
    (None, None)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_full_*.json")), key=os.path.getmtime)
    unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for f in reversed(files):
        try:
            with open(f) as fh:
                cap = json.load(fh)
        except Exception:
            continue
        for name, d in cap.get("kernels", {}).items():
            if name.startswith(KPREFIX.get(cls, "?")):
                tot = 0.0
                for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    v, u = (d.get(key, "0 byte").split() + ["byte"])[:2]
                    tot += float(v) * unit.get(u, 1.0)
                return tot, f"{os.path.relpath(f, ROOT)}: {name}, one launch (grid {d.get('launch__grid_size')})"
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

def solve_level_roofline(sol_roof, pk):
    """Roofline object on the paper's algorithmic flops for a whole solve (used for C4's lanes)."""
    f = sol_roof.get("frac_of_fp32_fp64_roofline")
    return {"bound": "fp32-simt+fp64-tensor", "kernel": "whole mp_orth solve (all kernels)",
            "achieved": sol_roof["gflops"] / 1e3, "peak": None, "unit": "TFLOP/s", "frac": f, "traffic": None,
            "algorithmic": "costmodel.flops (paper Table 3): low 25a+b fp32 on FFMA, high 6a+(4+3k)b fp64 on DMMA; "
                           "frac = (low/P32 + high/P64) / measured time",
            "peak_source": "measured live by sylv_microbench"}


def phase_rooflines(pk, kind, m, n, k, cx, rep, kern):
    """Per phase of one solve, on SURVEY.md 8(d)'s algorithmic flops (a = m^3+n^3, b = mn(m+n); Lyapunov:
    one n^3 Schur), against the live FFMA / DMMA peaks:
      schur    25 a fp32 flops (Hessenberg + QR sweeps + Schur vectors) / the Schur-pair wall time;
      gemm     6 a + (4+2k) b fp64 flops (orthonormalisation, S_A, S_B, F, k residuals, recovery) / the
               summed DMMA kernel time of the step (event-timed per launch);
      trsyl    (1+k) b flops (Y0 in fp32 + k corrections) / the summed trsyl kernel time."""
    mult = 4.0 if cx else 1.0
    a = float(n ** 3) if kind == "lyapunov" else float(m ** 3 + n ** 3)
    b = float(m * n * (m + n))
    out = {}

    def put(name, flops, ms, peak_key, note):
        if not ms:
            return
        tf = flops / (ms * 1e-3) / 1e12
        pkv = pk.get(peak_key)
        out[name] = {"flops": flops, "ms": ms, "tflops": tf, "peak": pkv, "peak_kind": peak_key,
                     "frac": tf / pkv if pkv else None, "flop_model": note}

    put("schur", mult * 25.0 * a, rep.ms_schur, "ffma", "25a fp32 (paper Table 3 low-precision Schur)")
    dm = (kern or {}).get(KCLASSES[0], {})
    put("gemm_fp64", mult * (6.0 * a + (4.0 + 2.0 * k) * b), dm.get("ms_per_step"), "dmma",
        "6a+(4+2k)b fp64 (GEMM-shaped high-precision flops)")
    tr = (kern or {}).get(KCLASSES[4], {})
    put("trsyl", mult * (1.0 + k) * b, tr.get("ms_per_step"), "ffma",
        "(1+k) b: Y0 + k corrections, mn(m+n) each (peak shown: FFMA; the corrections run in fp64)")
    return out


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
        return M.solve(A, B, C, kind=pr.kind, variant=args.variant, out=X, correction_bits=args.correction)

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
            Xe, _ = M.solve(dA, dB, dC, kind=pr.kind, variant=args.variant, correction_bits=args.correction)
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
    # ---- rooflines: per phase on the paper's algorithmic flops (headline: the dominant Schur phase) ----
    roof = sol_roof = kern = gemm_roof = phases = None
    if rank == 0:
        gemm_roof, pk = dmma_roofline(L, st, dev, m)
        _, kern = kernel_rooflines(krows, pk, args.steps)
        dm = kern.get(KCLASSES[0])
        if dm and "tflops" in dm:  # the north star's "FP64 tensor peak in its GEMM phases", live in the step
            gemm_roof["in_step"] = {"tflops": dm["tflops"], "frac": dm.get("frac_of_peak"),
                                    "ms_per_step": dm["ms_per_step"]}
        sol_roof = solve_roofline(pk, args.variant, pr.kind, m, n, k, cx, total_ms / args.steps / 1e3, 1)
        sol_roof["phase_ms"] = {"schur": reps[-1].ms_schur, "orth": reps[-1].ms_orth, "setup": reps[-1].ms_setup,
                                "y0": reps[-1].ms_y0, "refine": reps[-1].ms_refine, "recover": reps[-1].ms_recover}
        phases = phase_rooflines(pk, pr.kind, m, n, k, cx, reps[-1], kern)
        sch = phases.get("schur")
        if sch and args.variant != "bs":
            traffic, tsrc = ncu_traffic(3)
            roof = {"bound": "fp32-simt", "kernel": ("Schur phase: hess_panel2 + chase2 + apply_z_far/cl + schur_mss "
                                                     "kernels (the dominant phase of the step)"),
                    "achieved": sch["tflops"], "peak": sch["peak"], "unit": "TFLOP/s", "frac": sch["frac"],
                    "traffic": traffic, "traffic_source": tsrc,
                    "share_of_step": reps[-1].ms_schur / (total_ms / args.steps),
                    "algorithmic": (f"25(m^3+n^3) = {sch['flops']:.3e} fp32 flops per solve (SURVEY.md 8d) / the "
                                    f"Schur-pair wall time {sch['ms']:.1f} ms (CUDA events on the solve stream)"),
                    "peak_source": "FFMA peak measured live by sylv_microbench (MEASURED_PEAKS.json has no fp32)"}
        else:
            roof = dict(gemm_roof)
    # ---- CPU baseline (rank 0 at N=1): the Python reference at C0, else the oracle port, all host threads ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.config == "c0":
            cpu = cpu_baseline_python("c0", m, n)
        if cpu is None:
            cpu = cpu_baseline_oracle(min(args.cpu_sample_m, m), m, n, config=args.config)
    # ---- C4 sharded batch beside the headline (all ranks; strong scaling over the N GPUs) ----
    c4 = None
    if args.config == "ch" and args.variant != "bs" and not args.no_c4:
        r4 = measure_c4(args, rank, world, dev, max(2, min(args.steps, 3)), 2, with_kernels=False)
        c4 = {"metric": f"mixed-precision Sylvester solves/sec (c4: {r4['total']} equations, m=n={r4['m']})",
              "value": r4["value"], "unit": "solves/s", "ms_per_step": r4["ms_per_step"], "scaling": "strong",
              "per_rank": r4["per_rank"], "iterations": r4["ks"], "failed": r4["failed"],
              "max_backward_error": r4["max_backward_error"], "e2e": r4["e2e"], "gpu_launches": r4["launches"],
              "workload": "512 independent config-0 equations sharded by index over the ranks + gather of X"}
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
                       "correction_bits": args.correction,
                       "converged": all(bool(r.converged) and r.status == 0 for r in reps),
                       "parallelism": f"replicas x{world}"},
            "roofline": roof, "phase_rooflines": phases, "gemm_phase_roofline": gemm_roof,
            "kernels_impl_flops": kern, "solve_roofline": sol_roof,
            "cpu_baseline": cpu, "e2e": e2e, "c4_batch": c4,
            "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
            "gpu_launches": int(launches),
            "measured_peaks": {"hbm_gbs": peaks.get("hbm_gbs"), "bf16_tflops": peaks.get("bf16_tflops")},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
def measure_c4(args, rank, world, dev, steps, warmup, with_kernels=True):
    """C4: `batch` independent equations (config-0 recipe, m=n=512, entropy seed+i), sharded by equation
    index over the ranks; each rank solves its block with the lane executor (sylv_solve_batched), then one
    gather of X to rank 0 (the only collective), inside the timed region.  Total work is fixed as N grows:
    scaling "strong".  Returns a dict of measurements (max over ranks)."""
    import torch
    import torch.distributed as dist
    import paper_2503_03456_b200 as M
    from paper_2503_03456_b200 import _native, problems as P
    from paper_2503_03456_b200.batch import gather_solutions, shard_range
    L = _native.lib()
    m = args.m if (args.m and args.config == "c4") else P.FULL_SIZES["c4"][0]
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
        _, reps = M.solve_batched(A, B, C, out=X, lanes=args.lanes, correction_bits=args.correction)
        if world > 1:
            gather_solutions(X, total)
        return reps

    for _ in range(warmup):
        reps = step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    launches0 = L.sylv_launch_count()
    with ClockSampler(dev.index) as clk:
        for i in range(steps):
            flush.fill_(float(i))
            evs[i][0].record(st)
            reps = step()
            evs[i][1].record(st)
        torch.cuda.synchronize(dev)
    launches = (L.sylv_launch_count() - launches0) // max(1, steps)
    krows = None
    if with_kernels:
        ktimer(L, 1)  # per-kernel-class event timing over a repetition of the timed steps
        for i in range(steps):
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
    value = steps * total / (total_ms / 1e3)
    ks = sorted({r.iterations for r in reps})
    st_bad = sum(1 for r in reps if r.status != 0)
    be = max(r.backward_error for r in reps)
    e2e = None
    if not args.no_e2e:  # pinned host inputs -> device, batched solve, X -> host, gather
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for i in range(max(1, steps)):
            flush.fill_(float(i))
            e0.record(st)
            A.copy_(hA, non_blocking=True)
            B.copy_(hB, non_blocking=True)
            C.copy_(hC, non_blocking=True)
            M.solve_batched(A, B, C, out=X, lanes=args.lanes, correction_bits=args.correction)
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
        e2e = {"value": max(1, steps) * total / (tot / 1e3), "unit": "solves/s",
               "h2d_bytes_per_step": cnt * 3 * m * m * es, "d2h_bytes_per_step": cnt * m * m * es}
    return dict(value=value, ms_per_step=total_ms / steps, m=m, total=total, per_rank=cnt, ks=ks, failed=st_bad,
                max_backward_error=be, e2e=e2e, launches=int(launches), krows=krows, clk=clk, reps=reps)


def run_c4(args):
    """--config c4: the sharded batch as the line's own workload."""
    import torch
    import torch.distributed as dist
    rank, local, world = dist_info()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2503_03456_b200 import _native
    L = _native.lib()
    peaks = measured_peaks()
    r = measure_c4(args, rank, world, dev, args.steps, args.warmup)
    m, total = r["m"], r["total"]
    if rank == 0:
        st = torch.cuda.current_stream(dev)
        gemm_roof, pk = dmma_roofline(L, st, dev, m)
        _, kern = kernel_rooflines(r["krows"], pk, args.steps)
        # 64 concurrent lanes: per-launch event intervals include queueing behind the other lanes'
        # kernels, so they cannot give a per-kernel rate; the roofline object is the solve-level
        # algorithmic-flop roofline and the DMMA engine timed alone on the same GEMM shape
        sol_roof = solve_roofline(pk, "orth", "general", m, m, max(r["ks"]), False, r["ms_per_step"] / 1e3,
                                  r["per_rank"])
        roof = solve_level_roofline(sol_roof, pk)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline_oracle(m, m, m, config="c0")
        clocks = r["clk"].summary()
        reps = r["reps"]
        line = {
            "metric": f"mixed-precision Sylvester solves/sec (c4: {total} equations, m=n={m})",
            "value": r["value"], "unit": "solves/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic (seeded Philox, entropy seed+index)",
            "config": {"workload": f"c4: {total} x real general m=n={m}, mp_orth binary32/binary64, the whole "
                                   f"batch per step, sharded by equation index + gather of X to rank 0",
                       "m": m, "n": m, "batch": total, "per_rank": r["per_rank"], "lanes": args.lanes or 64,
                       "correction_bits": args.correction,
                       "iterations": r["ks"], "failed": r["failed"], "max_backward_error": r["max_backward_error"],
                       "lane_phase_ms_mean": {f: round(sum(getattr(x, "ms_" + f) for x in reps) / len(reps), 2)
                                              for f in ("schur", "orth", "setup", "y0", "refine", "recover",
                                                        "total")},
                       "l2": "flushed between steps (256 MiB write); per-rank working set >> 126 MB L2",
                       "parallelism": f"shard x{world} + gather"},
            "roofline": roof, "gemm_phase_roofline": gemm_roof, "kernels": kern, "solve_roofline": sol_roof,
            "cpu_baseline": cpu, "e2e": r["e2e"],
            "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
            "gpu_launches": r["launches"],
            "measured_peaks": {"hbm_gbs": peaks.get("hbm_gbs"), "bf16_tflops": peaks.get("bf16_tflops")},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def self_launch(args):
    """`python bench.py --gpus N` outside torchrun: re-run under torch.distributed.run with N ranks."""
    import random
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(random.randint(20000, 40000)),
           os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        self_launch(args)
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c4":
        run_c4(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
