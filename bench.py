#!/usr/bin/env python
"""bench.py — emRKC node-steps/s (fp64) on B200, BASELINE.json's metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config WORKLOAD]

A step is one emRKC time step (P/src/multirate.cpp:173-189) of the whole
workload grid; node-steps/s = nodes x steps / seconds. Defaults: N = 1, the
largest single-GPU configuration of BASELINE.json: config 4's grid
(512x512x256 = 67M nodes, h 0.1 mm, sigma (0.3, 0.1, 0.1), dt 0.05 ms; HH
stands in for the absent TTP model, s = 1, m = 2; the simulation hits the
reference's own NumericalAbort at step 65, so timed repeats stop there),
W = 5, K = 100. BASELINE configs[1] (128^3) and configs[0] (2-D 256^2) are
`also` lines.

`value`  : device time (CUDA events, per kernel launch, on the launching
           stream) with the state resident in HBM; L2 (126 MB) is flushed
           before every timed step, outside the timed pairs, by a 256 MiB
           memset followed by a 256 MiB read pass (so the memset's dirty
           lines are written back before the step, not during it).
`e2e`    : the per-call drop-in (emrkc_step_host: pinned host state in,
           one device step, host state out), wall clock around each call.
`roofline`: the step's dominant kernel, algorithmic bytes / its mean launch
           time against MEASURED_PEAKS.json hbm_gbs.
`cpu_baseline`: the reference's own code (oracle/_ref, compiled from the
           reference sources) on 1 host core, bounded sample (the grid's
           central 16-plane slab when a full step takes minutes), stepping
           loop only (the reference's wall_time window,
           P/src/simulate.cpp:175,230).
`--impl reference`: the reference CPU implementation on all usable host
           cores (independent replicas: the reference has no intra-run
           parallelism, P/src/experiments.cpp:22-37), same sample, W warm-up
           and K timed steps per replica; never maps the product library.
Multi-GPU (torchrun, one process per GPU): the grid is split into z-slabs
(strong scaling) and V halo planes go to the neighbours by peer stores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

FLUSH_BYTES = 256 << 20  # > 2x the 126 MB L2
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_traffic.json")

# Algorithmic bytes per node of each kernel launch: the fp64
# fields a launch must read and write at least once.
KERNEL_BYTES = {
    ("m1", "first_outer"): 64,   # g_{j-1} in (4 fields), g_j out (4)
    ("m1", "outer"): 96,         # + g_{j-2} in
    ("first", "first_outer"): 64,  # g_{j-1} in (4); gates of g_j (3) + d_1 out
    ("first", "outer"): 88,        # + gates of g_{j-2}... (V of g_{j-2} read later)
    ("tb", "first_outer"): 24,     # k_vin_tb: d_1, V of g_{j-1} in; V of g_j out
    ("tb", "outer"): 32,           # + V of g_{j-2}
    ("tb_skip", None): 0,          # stages 3..m ran inside the k = 2 launch
    ("inner2", None): 16,        # d_1 in, d_2 out
    ("inner", None): 32,         # d_{k-1}, d_{k-2}, d_1 in; d_k out
    ("last2", "first_outer"): 24,  # d_1, V of g_{j-1} in; V of g_j out
    ("last2", "outer"): 32,        # + V of g_{j-2}
    ("last", "first_outer"): 40,   # d_{m-1}, d_{m-2}, d_1, V in; V out
    ("last", "outer"): 48,
    ("fused", "first_outer"): 64,  # k_fused2: g_0 in (4 fields), g_1 out (4); d_1 stays on chip
    ("fused_skip", None): 0,       # level 2 ran inside the fused launch
    ("xstep", "first_outer"): 64,  # k_step_x: inner stage 2 of step n + node update of step n + 1
    ("x_first", "first_outer"): 0,  # the node level as its own launch: first step of a run only
    ("zpipe", "first_outer"): 64,  # the whole z-pipelined step (node + inner chunks, 2 streams)
    ("zpipe_skip", None): 0,       # timed inside the step's event pair
}
KERNEL_ROLES = {"m1": ("node", "m = 1: whole outer stage"),
                "first": ("node", "m >= 2: ionic + inner stage 1"),
                "inner2": ("vin", "inner stage 2"), "inner": ("vin", "inner stage k"),
                "last2": ("vin", "last inner stage, m = 2"),
                "last": ("vin", "last inner stage"),
                "tb": ("vin", "inner stages 2..m, temporally blocked"),
                "tb_skip": ("vin", "fused into the k = 2 launch"),
                "fused": ("fused2", "s = 1, m = 2: node update + inner stage 2 + outer update "
                                    "in one persistent pass"),
                "fused_skip": ("fused2", "level 2 ran inside the fused launch"),
                "zpipe": ("zpipe", "s = 1: node-kernel z-chunks overlapped with the inner-stage "
                                   "chunks on a second stream (one event pair per step)"),
                "zpipe_skip": ("zpipe", "timed with the step"),
                "xstep": ("xstep", "s = 1, m = 2: inner stage 2 of step n + ionic update and inner "
                                   "stage 1 of step n + 1 in one launch (cross-step fusion)"),
                "x_first": ("node", "m >= 2: ionic + inner stage 1 (first step of the run only)")}


def kernel_name(kind: str, problem, node_kernel: int = 0) -> str:
    """Kernel family the library selects (emrkc_capi.cpp init_handle):
    EMRKC_PIPE 3 (default; TMA, needs n0 even and dim >= 2), 1 (cp.async),
    2 (persistent node kernel), 0 (z-march)."""
    pipe = int(os.environ.get("EMRKC_PIPE") or 3)
    if pipe == 3 and (problem.dim < 2 or int(problem.n[0]) % 2):
        pipe = 1
    if problem.dim < 2:
        pipe = 0
    role, what = KERNEL_ROLES[kind]
    if role == "fused2":
        return f"k_fused2 ({what})"
    if role == "xstep":
        return f"k_step_x ({what})"
    if role == "zpipe":
        return f"k_node_tma + k_vin_tma_r z-pipelined step ({what})"
    fam = {3: "tma", 1: "pipe", 2: "persist" if role == "node" else "pipe", 0: "fast"}[pipe]
    if kind.startswith("tb"):
        fam = "tb"
    if role == "node" and node_kernel == 1:  # emrkc_node_kernel: pair-per-thread node kernel
        fam = "pair"
    return f"k_{role}_{fam} ({what})"


def tb_active(problem, m: int) -> bool:
    """k_vin_tb runs stages 2..m (emrkc_capi.cpp use_tb): 3-D whole grid on
    the TMA path, 2 <= m - 1 <= 4 (default; EMRKC_TB=0 disables)."""
    pipe = int(os.environ.get("EMRKC_PIPE") or 3)
    return (problem.dim == 3 and pipe == 3 and int(problem.n[0]) % 2 == 0
            and int(os.environ.get("EMRKC_TB") or 1) != 0 and 2 <= m - 1 <= 4)


def launch_kinds(s: int, m: int, problem=None, fused: int = 0):
    """(kind, outer) of each launch of one step, in launch order
    (emrkc_fused_active: 1 = the s = 1, m = 2 step as one k_fused2 pass,
    2 = the z-pipelined step, timed as one unit)."""
    if fused == 1:
        return [("fused", "first_outer"), ("fused_skip", None)]
    if fused == 2:
        return [("zpipe", "first_outer")] + [("zpipe_skip", None)] * (s * m - 1)
    if fused == 3:
        return [("x_first", "first_outer"), ("xstep", "first_outer")]
    out = []
    tb = problem is not None and tb_active(problem, m)
    for j in range(1, s + 1):
        o = "first_outer" if j == 1 else "outer"
        for k in range(1, m + 1):
            if m == 1:
                out.append(("m1", o))
            elif k == 1:
                out.append(("first", o))
            elif tb:
                out.append(("tb", o) if k == 2 else ("tb_skip", None))
            elif k < m:
                out.append(("inner2" if k == 2 else "inner", None))
            else:
                out.append(("last2" if m == 2 else "last", o))
    return out


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region (NVML,
    every ~5 ms; nvidia-smi as a fallback)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index: int, period_s: float = 0.005):
        self.idx = gpu_index
        self.period = period_s
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._th = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None
            self.max_mhz = None

    def _sample(self):
        if self._nvml is not None:
            nv = self._nvml
            sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
            try:
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
            return (float(sm), float(self.max_mhz), int(rs))
        out = subprocess.run(["nvidia-smi", "-i", str(self.idx),
                              "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5)
        a = [x.strip() for x in out.stdout.strip().split(",")]
        return (float(a[0]), float(a[1]), int(a[2], 16))

    def _poll(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._th = threading.Thread(target=self._poll, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"],
                    "samples": 0}
        busy = [s for s in self.samples if not (s[2] & 0x1)] or self.samples  # drop GpuIdle
        reasons = set()
        for s in busy:
            for bit, name in self.REASONS.items():
                if s[2] & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in busy),
                "sm_max_mhz": max(s[1] for s in busy), "reasons": sorted(reasons),
                "samples": len(busy), "source": "nvml" if self._nvml else "nvidia-smi"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def ncu_traffic(workload: str):
    try:
        with open(PROFILE_SUMMARY) as f:
            d = json.load(f)
        return d.get(workload)
    except Exception:
        return None


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# CPU legs (the oracle is only ever the checker / the reported baseline)
# ---------------------------------------------------------------------------

def cpu_impl():
    from oracle.oracle import Oracle, Reference, have_reference

    if have_reference():
        return Reference(), "reference"
    return Oracle(), "port"


# Bounded CPU sample of a large grid: its central SAMPLE_DEPTH planes as a
# standalone no-flux slab (workloads.z_slab_sample). A full step of config
# 4's grid takes ~40 s on one core; the 512x512x16 slab takes ~2.5 s and
# holds the centre stimulus.
SAMPLE_DEPTH = 16
SAMPLE_MIN_NODES = 4_500_000


def cpu_sample(w, resting):
    """(workload, y0, label) the CPU legs time: the whole grid when it is
    small, else the central z-slab (same per-node work)."""
    from paper_2401_01745_b200 import workloads

    p = w.problem
    if p.dim == 3 and w.n_nodes > SAMPLE_MIN_NODES:
        nz = int(p.n[2])
        z0 = max(0, nz // 2 - SAMPLE_DEPTH // 2)
        ws, ys = workloads.z_slab_sample(w, z0, SAMPLE_DEPTH, resting=resting)
        return ws, ys, (f"central slab z {z0}..{z0 + SAMPLE_DEPTH - 1} of {w.name} "
                        f"({int(p.n[0])}x{int(p.n[1])}x{SAMPLE_DEPTH} = {ws.n_nodes} nodes, "
                        f"standalone no-flux problem, rho estimated on it)")
    return w, w.initial_state(resting=resting), f"the full {w.name} grid"


def product_lib_mapped() -> bool:
    """Whether this process has the product library mapped (the CPU arm
    must not)."""
    try:
        with open("/proc/self/maps") as f:
            return "libemrkc_b200" in f.read()
    except OSError:
        return False


def cpu_baseline(w, budget_s=15.0):
    """The reference's stepping loop on ONE host core over a bounded sample
    of the workload (~budget_s of stepping), its own rho estimates."""
    impl, kind = cpu_impl()
    ws, y0, label = cpu_sample(w, impl.resting_state)
    p = ws.problem
    rF = impl.estimate_rho(p, 0, 0.0, y0)[0].rho
    rS = ws.rho_S_forced if ws.rho_S_forced is not None else impl.estimate_rho(p, 1, 0.0, y0)[0].rho
    _, _, t1 = impl.run(p, y0, 0, 1, ws.dt, ws.eps, rF, rS)
    k = int(max(1, min(w.n_steps, budget_s / max(t1, 1e-6))))
    _, res, wall = impl.run(p, y0, 0, k, ws.dt, ws.eps, rF, rS)
    v = ws.n_nodes * res.steps_done / wall if wall > 0 else None
    return {"value": v, "unit": "node-steps/s", "cores": 1, "kind": kind,
            "sample": f"{res.steps_done} emRKC steps of {label} from the seeded initial state, "
                      f"1 thread, stepping loop wall time {wall:.2f} s "
                      f"({'oracle/_ref: reference sources, -O3' if kind == 'reference' else 'oracle/emrkc_oracle.c'}); "
                      f"plan s={res.s} m={res.m}"}


REF_BUDGET_S = 200.0  # wall budget of the reference arm's timed steps


def reference_arm(args, w):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference sources; the C restatement if they are absent) on all usable
    host cores as independent concurrent replicas (the reference has no
    intra-run parallelism; its only pool is over independent experiment
    cells, P/src/experiments.cpp:22-37). Each replica runs W warm-up steps,
    then K timed steps of the bounded sample (cpu_sample), stepping loop
    only (the reference's wall_time window, P/src/simulate.cpp:175,230).
    This process never maps the product library: the initial state uses
    the reference's own resting_state."""
    ws_, rank, _ = dist_env()
    if rank != 0:
        return 0
    impl, kind = cpu_impl()
    ws, y0, label = cpu_sample(w, impl.resting_state)
    p = ws.problem
    rF = impl.estimate_rho(p, 0, 0.0, y0)[0].rho
    rS = ws.rho_S_forced if ws.rho_S_forced is not None else impl.estimate_rho(p, 1, 0.0, y0)[0].rho
    cores = cpu_count()
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    per_replica = 24 * 8 * p.state_len()  # the reference's per-call Vec temporaries
    threads = int(max(1, min(cores, avail * 0.6 // per_replica)))
    _, _, t1 = impl.run(p, y0, 0, 1, ws.dt, ws.eps, rF, rS)
    k = int(args.steps)
    capped = ""
    if k * t1 * 1.15 > REF_BUDGET_S:
        k = int(max(1, REF_BUDGET_S / (1.15 * t1)))
        capped = f"; K capped from {args.steps} to {k} steps (wall budget {REF_BUDGET_S:.0f} s)"
    if kind == "reference":
        impl.bench(p, y0, args.warmup, ws.dt, ws.eps, rF, rS, threads)  # warm-up
        secs = impl.bench(p, y0, k, ws.dt, ws.eps, rF, rS, threads)
        wall = float(np.max(secs))
    else:
        threads = 1
        impl.run(p, y0, 0, args.warmup, ws.dt, ws.eps, rF, rS)
        _, _, wall = impl.run(p, y0, 0, k, ws.dt, ws.eps, rF, rS)
    v = threads * ws.n_nodes * k / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "node-steps/s",
        "n_gpus": ws_, "steps": k, "warmup": args.warmup, "ms_per_step": wall * 1e3 / k,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded HH resting state + noise)", "config": config_of(w, ws_),
        "cpu_baseline": {"value": v, "unit": "node-steps/s", "cores": threads, "kind": kind,
                         "sample": f"{threads} concurrent independent replicas x {k} emRKC steps of "
                                   f"{label} (the reference's serial loop per replica, "
                                   f"{args.warmup} warm-up steps each){capped}; 1-thread step "
                                   f"{t1:.3f} s"},
        "e2e": {"value": v, "unit": "node-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_lib_mapped": product_lib_mapped(),
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "emRKC node-steps/s (fp64)"
# N = 1 headline: the largest single-GPU configuration of BASELINE.json,
# config 4's grid (512x512x256, 67M nodes; HH stands in for the absent TTP
# model, SURVEY §8(c) option 1).
HEADLINE = "hh3d_512x512x256"


def config_of(w, n_gpus):
    d = w.describe()
    d["parallelism"] = f"z-slab x{n_gpus}" if n_gpus > 1 else "single GPU"
    d["l2"] = ("flushed before every timed step: 256 MiB memset, then a 256 MiB read pass "
               "(dirty lines written back outside the timed pairs)")
    return d


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def measure_device(w, device, warmup, steps, with_e2e=True, clocks=None, ramp_s=0.3, rho=None):
    """Device-resident timing of one workload on one GPU.

    Warm-up: `warmup` steps, then untimed steps until `ramp_s` of GPU work
    has passed (SM clock ramp). Timed: `steps` steps as back-to-back
    repeats of the workload's own simulation (each repeat restarts from the
    seeded initial state at t = 0 and runs at most the workload's step count),
    every kernel launch timed by its own CUDA-event pair, L2 flushed before
    every step outside the pairs. `clocks` (a ClockSampler) is active over
    the timed loop only."""
    import ctypes as C

    from paper_2401_01745_b200 import capi
    from paper_2401_01745_b200.capi import RunResult, dptr
    from paper_2401_01745_b200.monodomain import MonodomainOperator

    lib = capi.load()
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p, device)
    op.set_state(y0)
    if rho is not None:
        rF, rS = rho
    else:
        rF = op.estimate_spectral_radius(capi.EMRKC_RHS_F, 0.0).rho
        rS = w.rho_S_forced if w.rho_S_forced is not None else \
            op.estimate_spectral_radius(capi.EMRKC_RHS_S, 0.0).rho
    rep = capi.StepReport()
    lib.emrkc_plan_step(w.dt, rF, rS, w.eps, C.byref(rep))
    per = rep.s * rep.m
    op.run(0, warmup, w.dt, rF, rS, w.eps)
    t0 = time.perf_counter()
    ramp = 0
    while time.perf_counter() - t0 < ramp_s:
        op.run(0, max(1, min(50, w.n_steps)), w.dt, rF, rS, w.eps)
        op.set_state(y0)
        ramp += 1
    # a simulation that hits NumericalAbort / the norm guard at step kr is
    # timed over its first kr steps only (later steps would only run the
    # kernels' skip path and inflate the rate)
    op.set_state(y0)
    rr = op.run(0, w.n_steps, w.dt, rF, rS, w.eps)
    kr = max(1, int(rr.abort_step)) if rr.aborted else w.n_steps
    chunks = []
    left = steps
    while left > 0:
        chunks.append(min(left, kr))
        left -= chunks[-1]
    launch_ms = np.zeros(steps * per)
    results = []
    ctx = clocks if clocks is not None else _Null()
    with ctx:
        off = 0
        for ck in chunks:
            op.set_state(y0)
            res = RunResult()
            rc = lib.emrkc_run_timed(op.handle, 0, ck, w.dt, w.eps, 0, rF, rS, FLUSH_BYTES,
                                     dptr(launch_ms[off:]), ck * per, C.byref(res))
            if rc:
                raise RuntimeError(lib.emrkc_last_error(op.handle).decode())
            results.append(res)
            off += ck * per
    # the workload's whole simulation through emrkc_run (run_simulation's
    # loop; small grids take the one-launch resident kernel), device events
    # around the run, no L2 flush between its steps
    # (a run that aborts is timed over the steps before the abort only)
    run = None
    if kr >= 2:
        run_ms = []
        for _ in range(3):
            op.set_state(y0)
            rr = op.run(0, kr, w.dt, rF, rS, w.eps)
            run_ms.append(rr.device_ms)
        run = {"value": w.n_nodes * kr / (min(run_ms) * 1e-3), "unit": "node-steps/s",
               "ms_per_step": min(run_ms) / kr, "steps": kr,
               "note": "emrkc_run of the simulation" +
                       (f" up to its NumericalAbort/guard at step {kr}" if kr < w.n_steps else "") +
                       ", best of 3, device time of the run, no L2 flush between steps"}
    out = {"op": op, "y0": y0, "rF": rF, "rS": rS, "s": rep.s, "m": rep.m, "run": run,
           "fused": int(lib.emrkc_fused_active(op.handle)),
           "node_kernel": int(lib.emrkc_node_kernel(op.handle)),
           "launch_ms": launch_ms.reshape(steps, per), "res": results[-1], "steps": steps,
           "repeats": len(chunks), "aborted": any(r.aborted for r in results),
           "abort_at": kr if kr < w.n_steps else None}
    if with_e2e:
        out["e2e"] = measure_e2e(op, w, y0, rF, rS, min(steps, 20))
        out["e2e_run"] = measure_e2e_run(op, w, y0, rF, rS)
    return out


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def measure_e2e(op, w, y0, rF, rS, k):
    """Per-call drop-in: pinned host y in -> device step -> host y out."""
    import ctypes as C

    import torch

    from paper_2401_01745_b200 import capi

    lib = capi.load()
    n = y0.size
    hin = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hout = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hin.numpy()[:] = y0
    pin = C.cast(hin.data_ptr(), capi.DP)
    pout = C.cast(hout.data_ptr(), capi.DP)
    rep = capi.StepReport()
    # warm-up call
    lib.emrkc_step_host(op.handle, 0.0, pin, pout, n, w.dt, w.eps, 0, rF, rS, C.byref(rep))
    t0 = time.perf_counter()
    for r in range(k):
        rc = lib.emrkc_step_host(op.handle, r * w.dt, pin, pout, n, w.dt, w.eps, 0, rF, rS,
                                 C.byref(rep))
        if rc:
            raise RuntimeError(lib.emrkc_last_error(op.handle).decode())
        hin, hout = hout, hin  # next step consumes this step's result
        pin, pout = pout, pin
    wall = time.perf_counter() - t0
    return {"value": w.n_nodes * k / wall, "unit": "node-steps/s",
            "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
            "steps": k, "ms_per_step": wall * 1e3 / k,
            "api": "emrkc_step_host (C ABI; drop-in of Vec emrkc_step(t, y, dt, rhs, ...))"}


def measure_e2e_run(op, w, y0, rF, rS, reps=3):
    """run_simulation's loop through the public API with host state: pinned
    host y in (emrkc_set_state), the workload's whole simulation on the
    device (emrkc_run: per-step abort / guard / gate range kept on the
    device, the run record read back), host y out (emrkc_get_state); wall
    clock, best of `reps`."""
    import ctypes as C

    import torch

    from paper_2401_01745_b200 import capi

    lib = capi.load()
    n = y0.size
    hin = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hout = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hin.numpy()[:] = y0
    pin = C.cast(hin.data_ptr(), capi.DP)
    pout = C.cast(hout.data_ptr(), capi.DP)
    lib.emrkc_set_state(op.handle, pin, n)
    rr = op.run(0, w.n_steps, w.dt, rF, rS, w.eps)
    k = int(rr.abort_step) if rr.aborted else w.n_steps
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        if lib.emrkc_set_state(op.handle, pin, n):
            raise RuntimeError(lib.emrkc_last_error(op.handle).decode())
        op.run(0, k, w.dt, rF, rS, w.eps)
        if lib.emrkc_get_state(op.handle, pout, n):
            raise RuntimeError(lib.emrkc_last_error(op.handle).decode())
        wall = time.perf_counter() - t0
        best = wall if best is None else min(best, wall)
    return {"value": w.n_nodes * k / best, "unit": "node-steps/s", "steps": k,
            "ms_per_step": best * 1e3 / k,
            "h2d_bytes_per_step": 8 * n / k, "d2h_bytes_per_step": 8 * n / k,
            "api": "emrkc_set_state (pinned host) + emrkc_run (the whole simulation, "
                   "run_simulation's loop) + emrkc_get_state"}


def gpu_launches_per_step(m) -> int:
    """Kernel launches of one step: 1 (fused), K node chunks + K (m - 1)
    inner chunks (z-pipelined, EMRKC_ZPIPE=K), else s m."""
    if m["fused"] == 1:
        return 1
    if m["fused"] == 2:
        return int(os.environ.get("EMRKC_ZPIPE") or 0) * m["m"]  # read at handle creation
    if m["fused"] == 3:
        return 1  # k_step_x (plus one node launch and one inner-stage launch per run)
    return m["s"] * m["m"]


def kernel_bytes(kind, nf: int) -> float:
    """KERNEL_BYTES at a state of nf SoA fields: the node kinds move every
    field (16 B per field and node; the synthetic width stand-in's aux
    fields included), the inner-stage kinds touch V only."""
    kb = KERNEL_BYTES[kind]
    if kind[0] in ("m1", "first", "fused", "zpipe") and nf != 4:
        kb = kb * nf / 4
    return kb


def roofline_of(m, w, peak, peak_kind):
    per_pos = m["launch_ms"].mean(axis=0)
    kinds = launch_kinds(m["s"], m["m"], w.problem, m.get("fused", 0))
    dom = int(np.argmax(per_pos))
    nf = w.problem.n_fields
    kb = kernel_bytes(kinds[dom], nf)
    achieved = kb * w.n_nodes / (per_pos[dom] * 1e-3) / 1e9
    step_ms = m["launch_ms"].sum(axis=1).mean()
    step_gbs = 16 * nf * w.n_nodes / (step_ms * 1e-3) / 1e9
    traffic = ncu_traffic(w.name)
    return {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": traffic,
        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
        "kernel": kernel_name(kinds[dom][0], w.problem, m.get("node_kernel", 0)),
        "alg_bytes_per_node": kb, "mean_launch_ms": float(per_pos[dom]),
        "share_of_step": float(per_pos[dom] / per_pos.sum()),
        "step_alg_bytes_per_node": 16 * nf, "step_achieved_gbs": step_gbs,
        "step_frac": step_gbs / peak,
    }


def b200_arm(args, w):
    ws, rank, local = dist_env()
    if ws > 1 or os.environ.get("EMRKC_BENCH_DIST") == "1":  # 1-rank run of the N>1 arm (test)
        return b200_dist(args, w)
    import torch  # noqa: F401  (pinned host buffers for e2e)

    peak, peak_kind = hbm_peak()
    clk = ClockSampler(local)
    m = measure_device(w, local, args.warmup, args.steps, clocks=clk)
    clocks = clk.summary()
    res = m["res"]
    total_ms = float(m["launch_ms"].sum())
    value = w.n_nodes * args.steps / (total_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "node-steps/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded HH resting state + N(0, 0.1 mV) V noise)",
        "config": config_of(w, 1),
        "plan": {"s": m["s"], "m": m["m"], "rho_F": m["rF"], "rho_S": m["rS"],
                 "eta": res.eta, "aborted": bool(m["aborted"]),
                 "timed_repeats": m["repeats"],
                 "timed_note": f"{args.steps} timed steps = {m['repeats']} repeat(s) of the "
                               f"workload's simulation from the seeded state (<= {w.n_steps} steps each)" +
                               (f"; the simulation hits the reference's NumericalAbort/guard at step "
                                f"{m['abort_at']}, so each repeat stops there" if m.get("abort_at") else "")},
        "roofline": roofline_of(m, w, peak, peak_kind),
        "e2e": m["e2e"],
        "e2e_run": m["e2e_run"],
        "run": m["run"],
        "gpu_launches": int(args.steps * gpu_launches_per_step(m)),
        "clocks": clocks,
    }
    y0, rF, rS = m["y0"], m["rF"], m["rS"]
    from paper_2401_01745_b200.monodomain import MonodomainOperator

    m["op"].close()
    del m
    if not args.no_extra:
        also = []
        from paper_2401_01745_b200 import workloads

        # BASELINE configs[1] and [0]; configs 3 and 4 at their models' state
        # width (CRN 21, TTP 19 fields) through the SYNTHETIC width stand-in
        # (HH + passive aux variables, no physiology claim): per-node bytes
        # of 336 / 304 B. Their rho comes from the HH state of the same grid
        # (the aux rows' eigenvalues, |k_a| <= 0.01/ms, do not reach rho_S or
        # rho_F; the plan s, m is the same).
        hh_rho = {"hh3d_512x512x256_w19": (rF, rS) if w.name == "hh3d_512x512x256" else None}
        # config 3's grid with HH, and config 5's finest grid (N = 200, m = 4:
        # inner stages 2..4 in one temporally blocked pass, k_vin_tb)
        for name in ("hh3d_128x128x128", "hh2d_256x256", "hh3d_256x256x128", "hh3d_sweep_200",
                     "hh3d_512x512x256_w19", "hh3d_256x256x128_w21"):
            if name == w.name:
                continue
            wx = workloads.get(name)
            rho = hh_rho.get(name)
            if rho is None and name.endswith(("_w19", "_w21")):
                base = workloads.get(name.rsplit("_w", 1)[0])
                mb = MonodomainOperator(base.problem, local)
                mb.set_state(base.initial_state())
                rho = (mb.estimate_spectral_radius(0, 0.0).rho,
                       mb.estimate_spectral_radius(1, 0.0).rho)
                mb.close()
            mx = measure_device(wx, local, 3, 20, with_e2e=False, rho=rho)
            tot = float(mx["launch_ms"].sum())
            entry = {"workload": name, "value": wx.n_nodes * 20 / (tot * 1e-3),
                     "unit": "node-steps/s", "ms_per_step": tot / 20, "s": mx["s"],
                     "m": mx["m"], "state_fields": wx.problem.n_fields,
                     "roofline": roofline_of(mx, wx, peak, peak_kind), "run": mx["run"]}
            if wx.problem.n_aux:
                entry["note"] = wx.note
            also.append(entry)
            mx["op"].close()
        line["also"] = also
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    print(json.dumps(line), flush=True)
    return 0


def b200_dist(args, w):
    from paper_2401_01745_b200 import dist

    return dist.bench_main(args, w, METRIC, config_of, hbm_peak, ClockSampler)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default=HEADLINE)
    ap.add_argument("--no-extra", action="store_true", help="skip the 'also' workloads")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    from paper_2401_01745_b200 import workloads

    w = workloads.get(args.config)
    if args.impl == "reference":
        return reference_arm(args, w)
    return b200_arm(args, w)


if __name__ == "__main__":
    sys.exit(main())
