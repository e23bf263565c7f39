#!/usr/bin/env python
"""bench.py — qCH_eff hot paths on B200 (libqcheff, sm_100a).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--secondary all|none|npad60,npad4096,sweep,magnus4096]

Headline (BASELINE.json metric, configs[1]): Magnus time coarse-graining of a
driven 3-level transmon, 10^5 intervals per GPU, SECOND order, intervals/s.
N > 1 GPUs: weak scaling — every rank owns 10^5 contiguous intervals of one
global evolution; the ranks all-gather their block products (NCCL) for the
ordered product.  Secondary lines (N = 1, rank 0): NPAD configs 1, 3, 4 and
Magnus config 5 (sampled), each with its own roofline.

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events
on the launching stream (L2 flushed between steps by writing a 256 MiB
buffer, outside the events); barrier + synchronize around the timed region;
max over ranks.  ``e2e`` repeats the step through the public API from pinned
host buffers (H2D of the inputs + D2H of the trajectory inside the timing).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASELINE["metric"]
M_PER_GPU = 100_000
SUB = 4
T_PER_GPU = 100.0


# ---------------------------------------------------------------- helpers --

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6545.6), "MEASURED_PEAKS.json"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.tmp, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        self.tmp.flush()
        rows = []
        try:
            for line in Path(self.tmp.name).read_text().splitlines():
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        loaded = [v for v in sm if v > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


class L2Flusher:
    def __init__(self, torch):
        self.buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def __call__(self):
        self.buf.fill_(1.0)


def time_steps(torch, fn, steps, flush, world):
    """Per-step CUDA-event timing (current stream); returns list of ms."""
    import torch.distributed as dist

    out = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(steps):
        flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    return out


def sum_over_ranks(torch, value, world):
    if world == 1:
        return value
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(torch, value, world):
    if world == 1:
        return value
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def fp64_peaks(torch, lib_mod):
    """Live FP64 probes (DFMA pipe, DMMA tensor pipe) -> TFLOP/s."""
    import ctypes

    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    res = {}
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for kind, name, iters in ((0, "dfma", 2000), (1, "dmma", 4000)):
        fl = ctypes.c_double(0)
        best = 0.0
        for _ in range(4):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            lib_mod.load().qch_peak_kernel(kind, sms * 8, iters, ctypes.c_void_p(sink.data_ptr()), ctypes.byref(fl),
                                           lib_mod.stream_ptr())
            e.record()
            torch.cuda.synchronize()
            best = max(best, fl.value / (s.elapsed_time(e) * 1e-3) / 1e12)
        res[name] = best
    # cuBLAS zgemm (library reference point for the DMMA path)
    a = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda")
    b = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        torch.matmul(a, b)
    e.record()
    torch.cuda.synchronize()
    res["cublas_zgemm"] = 3 * 8 * 4096**3 / (s.elapsed_time(e) * 1e-3) / 1e12
    del a, b
    # cuBLASLt int8 (torch._int_mm, int32 accumulate) 8192^3: the measured
    # dense int8 tensor peak the Ozaki GEMM is held against (burst, best of 5)
    try:
        ia = torch.randint(-127, 128, (8192, 8192), dtype=torch.int8, device="cuda")
        ib = torch.randint(-127, 128, (8192, 8192), dtype=torch.int8, device="cuda")
        torch._int_mm(ia, ib.t())
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch._int_mm(ia, ib.t())
            e.record()
            torch.cuda.synchronize()
            best = max(best, 2.0 * 8192**3 / (s.elapsed_time(e) * 1e-3) / 1e12)
        res["cublaslt_int8_tops"] = best
        del ia, ib
    except Exception:  # pragma: no cover - no int8 GEMM in this torch build
        pass
    return res


def traffic_from_profiles(kernel: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        v = d.get(kernel)
        if isinstance(v, dict):
            return v.get("bytes_per_launch")
    return None


# ------------------------------------------------------- headline: Magnus --

def magnus_inputs(eff, world, rank):
    m = M_PER_GPU * world
    ch, grid = eff.driven_transmon(3, intervals=m, sub=SUB, t_final=T_PER_GPU * world)
    psi0 = np.array([1, 0, 0], dtype=np.complex128)
    return ch, grid, m, psi0


# Algorithmic FP64 flops per interval of the fused interval kernel (N=3, K=2,
# order 2): 17 complex N^3 GEMMs (8N^3 each) + 18 scale/add passes (4N^2) of
# the Taylor series (expm.py:66-68) + assembly of 1 + K + K(K+1)/2 operator
# terms (4N^2 each: real*complex + add) + second-order coefficients (~14*sub*K^2).
def magnus_flops_per_interval(n=3, k=2, sub=SUB):
    ncomm = k + k * (k - 1) // 2
    return 17 * 8 * n**3 + 18 * 4 * n * n + (1 + k + ncomm) * 4 * n * n + 14 * sub * k * k


# FP64 flops the fused kernel actually executes per interval (N=3, K=2,
# order 2, Taylor degree m = 7 for the config-2 norms): a^2 + m//2 Horner steps
# (27 complex MACs + 9 scalar-complex terms each), the lane run product and
# the warp scan (kR - 1 + 5 products per kR intervals), the trajectory
# mat-vec, assembly and coefficients.
def magnus_executed_flops_per_interval(n=3, k=2, sub=SUB, m=7, kr=2):
    mm = 8 * n**3
    ncomm = k + k * (k - 1) // 2
    return (mm + (m // 2) * (mm + 4 * n * n) + (kr - 1 + 5) * mm / kr + 8 * n * n
            + (1 + k + ncomm) * 4 * n * n + 14 * sub * k * k)


def cpu_magnus_sample(eff_models, n_int):
    """Oracle (numpy port of the reference, + 2nd order) on a bounded sample."""
    from oracle import magnus_oracle

    ch, grid = eff_models.driven_transmon(3, intervals=n_int, sub=SUB, t_final=T_PER_GPU * n_int / M_PER_GPU)
    d0 = ch.drift.data
    ctr = np.stack([c.data for c in ch.controls])
    psi0 = np.array([1, 0, 0], dtype=complex)
    t0 = time.perf_counter()
    magnus_oracle.evolve(d0, ctr, grid.signals, grid.t_start, grid.t_end, n_int, psi0, order=2)
    dt = time.perf_counter() - t0
    return n_int / dt, dt


def run_headline(torch, eff, lib, args, world, rank, local):
    from paper_2411_09982_b200 import magnus as mg
    from paper_2411_09982_b200 import sharding

    ch, grid, m, psi0 = magnus_inputs(eff, world, rank)
    psi0_dev = lib.to_device(psi0)
    flush = L2Flusher(torch)

    if world == 1:
        # the whole pipeline captured once as a CUDA graph; each step = 1 replay
        plan = mg.EvolvePlan(ch, grid, m, psi0, order=2, check=False)

        def step():
            plan.run()
    else:
        # interval sharding: per step pass 1 (fused kernel, prefix mode) ->
        # ONE NCCL all-gather of the N x N block products -> pass 2
        plan = sharding.ShardedEvolvePlan(ch, grid, m, psi0, order=2, check=False)

        def step():
            plan.run()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    lib.profile_read(reset=True)
    lib.profile_enable(True)
    n0 = lib.launch_count()
    with ClockSampler(local) as clk:
        ms = time_steps(torch, step, args.steps, flush, world)
    launches = lib.launch_count() - n0
    lib.profile_enable(False)
    prof = lib.profile_read(reset=True)
    plan.check()
    if world > 1:
        launches = 3 * args.steps  # fused (prefix mode) + apply_prefix + shard_traj per step
        # kernel timing pass: the step's halves are graph replays; time the
        # fused kernel (prefix mode) through eager launches of pass 1
        lib.profile_read(reset=True)
        lib.profile_enable(True)
        for _ in range(3):
            plan._prepare()
        torch.cuda.synchronize()
        lib.profile_enable(False)
        prof = lib.profile_read(reset=True)
    if world == 1:
        launches = 1 * args.steps  # graph replay = 1 libqcheff kernel (magnus_fused_kernel) per step
        # kernel timing pass (eager launches, CUDA events on the launching stream)
        lib.profile_read(reset=True)
        lib.profile_enable(True)
        for _ in range(3):
            mg.evolve_device(ch, grid, m, psi0_dev, check=False, order=2)
        lib.profile_enable(False)
        prof = lib.profile_read(reset=True)
    total_ms = max_over_ranks(torch, sum(ms), world)
    per_step = total_ms / args.steps
    value = M_PER_GPU * world / (per_step * 1e-3)

    # e2e through the public API (evolve) from pinned host buffers: every step
    # moves the control samples H2D and the trajectory D2H inside the timed
    # region (the problem objects are built once, as the reference arm's
    # timing excludes model construction too)
    sig_pinned = torch.empty(grid.signals.shape, dtype=torch.float64).pin_memory()
    sig_pinned.numpy()[:] = grid.signals
    ops = [ch.drift.data] + [c.data for c in ch.controls]
    chh = eff.ControlledHamiltonian(eff.HermitianOperator(ops[0], validate=False),
                                    [eff.HermitianOperator(o, validate=False) for o in ops[1:]])
    gh = eff.ControlGrid(grid.t_start, grid.t_end, sig_pinned.numpy())

    def e2e_step():
        if world == 1:
            tr = eff.evolve(chh, gh, m, psi0, order=2, check=False)
            return tr.amplitudes
        res = sharding.evolve_sharded(chh, gh, m, psi0, order=2, check=False)
        return res.trajectory.cpu().numpy()

    e2e_step()
    torch.cuda.synchronize()
    e2e_ms = time_steps(torch, e2e_step, max(3, args.steps), flush, world)
    e2e_per = max_over_ranks(torch, sum(e2e_ms), world) / len(e2e_ms)
    # the same with the plain (pageable) numpy signals a reference caller passes
    gp = eff.ControlGrid(grid.t_start, grid.t_end, np.array(grid.signals, copy=True))

    def e2e_pageable_step():
        if world == 1:
            return eff.evolve(chh, gp, m, psi0, order=2, check=False).amplitudes
        return sharding.evolve_sharded(chh, gp, m, psi0, order=2, check=False).trajectory.cpu().numpy()

    e2e_pageable_step()
    torch.cuda.synchronize()
    pg_ms = time_steps(torch, e2e_pageable_step, max(3, args.steps), flush, world)
    pg_per = max_over_ranks(torch, sum(pg_ms), world) / len(pg_ms)
    h2d = grid.signals.nbytes // world + sum(o.nbytes for o in ops) + psi0.nbytes
    d2h = (M_PER_GPU + 1) * 3 * 16

    k1 = prof.get("magnus_fused_kernel")
    roof = None
    if k1:
        k1_ms = k1[0] / k1[1]
        fl = magnus_flops_per_interval() * M_PER_GPU
        roof = {"kernel": "magnus_fused_kernel", "launch_ms": k1_ms, "flops_per_launch": fl,
                "executed_flops_per_launch": magnus_executed_flops_per_interval() * M_PER_GPU,
                "kernel_share_of_step": k1_ms / per_step}
    return dict(value=value, per_step=per_step, ms=ms, launches=launches // args.steps, clocks=clk.summary(),
                e2e=(M_PER_GPU * world / (e2e_per * 1e-3), h2d, d2h), e2e_pageable=M_PER_GPU * world / (pg_per * 1e-3),
                roof=roof, m=m)


# -------------------------------------------------------------- secondaries --

def _e2e_npad(torch, eff, h, reps, target=None, flush=lambda: None):
    """NPAD end to end through the public API: host numpy H -> HermitianOperator
    -> npad_run -> host diagonal (the reference contract, npad.py:320-354 +
    operators.py:120-131), H2D and D2H inside the timed region."""
    res = {}

    def step():
        st = eff.npad_run(eff.HermitianOperator(h), target, tol=1e-12)
        res["diag"] = st.current.diagonal()
        res["applied"] = st.applied

    step()
    ms = time_steps(torch, step, reps, flush, 1)
    per = sum(ms) / len(ms)
    return {"value": res["applied"] / (per * 1e-3), "unit": "rotations/s", "ms_per_solve": per,
            "h2d_bytes_per_step": int(h.nbytes), "d2h_bytes_per_step": int(res["diag"].nbytes),
            "path": "npad_run(HermitianOperator(host H)).current.diagonal() (pageable host H)"}


def sec_npad60(torch, eff, lib, args, peaks):
    from oracle import npad_oracle

    h = eff.transmon_resonator_hamiltonian(3, 20).data
    op = eff.HermitianOperator(h)
    op.device_tensor()
    op.max_abs()
    res = {}

    def step():
        res["st"] = eff.npad_run(op, tol=1e-12)

    for _ in range(3):
        step()
    lib.profile_read(reset=True)
    lib.profile_enable(True)
    ms = time_steps(torch, step, 10, lambda: None, 1)
    lib.profile_enable(False)
    prof = lib.profile_read(reset=True)
    rot = res["st"].applied
    per = sum(ms) / len(ms)
    kms = prof["npad_run_kernel"][0] / prof["npad_run_kernel"][1]
    e2e = _e2e_npad(torch, eff, h, 10)
    t0 = time.perf_counter()
    ref = npad_oracle.run_full_scan(h, tol=1e-12)
    cpu = ref["applied"] / (time.perf_counter() - t0)
    return {"workload": "config 1: NPAD transmon3 x resonator20 (dim 60), full diagonal, tol 1e-12",
            "metric": "NPAD rotations/s", "unit": "rotations/s", "value": rot / (per * 1e-3),
            "rotations": rot, "ms_per_solve": per, "us_per_rotation_kernel": kms * 1e3 / rot,
            "e2e": e2e,
            "roofline": {"bound": "latency", "note": "serial greedy chain; matrix resident in shared memory",
                         "achieved": 96 * 60 * rot / (kms * 1e-3) / 1e9, "peak": peaks[0], "unit": "GB/s",
                         "frac": 96 * 60 * rot / (kms * 1e-3) / 1e9 / peaks[0]},
            "cpu_baseline": {"value": cpu, "unit": "rotations/s", "cores": 1, "kind": "port",
                             "sample": "full solve (1022 rotations), oracle run_full_scan (reference algorithm)"}}


def sec_npad4096(torch, eff, lib, args, peaks, rotations=None):
    from oracle import npad_oracle

    n_q, n_r = 4, 1024
    h = eff.transmon_resonator_hamiltonian(n_q, n_r).data
    op = eff.HermitianOperator(h, validate=False)
    op.device_tensor()
    op.max_abs()
    res = {}
    mi = rotations

    def step():
        res["st"] = eff.npad_run(op, tol=1e-12, max_iter=mi)

    step()
    lib.profile_read(reset=True)
    lib.profile_enable(True)
    ms = time_steps(torch, step, 2, L2Flusher(torch), 1)
    lib.profile_enable(False)
    prof = lib.profile_read(reset=True)
    st = res["st"]
    per = sum(ms) / len(ms)
    kms = prof["npad_run_kernel"][0] / prof["npad_run_kernel"][1]
    n = n_q * n_r
    ach = 96 * n * st.applied / (kms * 1e-3) / 1e9
    e2e = _e2e_npad(torch, eff, h, 1, flush=L2Flusher(torch)) if not mi else None
    t0 = time.perf_counter()
    ref = npad_oracle.run_full_scan(h, tol=1e-12, max_iter=3)
    cpu = 3 / (time.perf_counter() - t0)
    return {"workload": f"config 3: NPAD transmon4 x resonator1024 (dim 4096) dense complex128, full diagonal, "
                        f"tol 1e-12, {'max_iter=' + str(mi) if mi else 'to convergence'}",
            "metric": "NPAD rotations/s", "unit": "rotations/s", "value": st.applied / (per * 1e-3),
            "rotations": st.applied, "converged": st.converged, "ms_per_solve": per,
            "us_per_rotation_kernel": kms * 1e3 / st.applied,
            "e2e": e2e,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peaks[0], "unit": "GB/s", "frac": ach / peaks[0],
                         "bytes_per_rotation": 96 * n, "note": "single greedy chain: latency-bound (see DESIGN.md)",
                         "traffic": (traffic_from_profiles("npad_coop_kernel@npad4096") or 0) / 2000 * st.applied
                         or None,
                         "traffic_note": "ncu DRAM bytes of a 2000-rotation launch (tools/prof_round.sh), scaled per "
                                         "rotation to this launch"},
            "cpu_baseline": {"value": cpu, "unit": "rotations/s", "cores": 1, "kind": "port",
                             "sample": "3 rotations of the same operator, oracle run_full_scan"}}


def sec_sweep(torch, eff, lib, args, peaks, world=1, rank=0, n_points=1024):
    """Config 4: 1024 (g, Delta) points of a dim-1024 transmon x resonator,
    subspace NPAD to convergence.  N > 1: the points are split in contiguous
    blocks over the ranks (sharding.sweep_sharded; strong scaling, no
    collective on the data path)."""
    from oracle import npad_oracle
    from paper_2411_09982_b200 import npad as npd
    from paper_2411_09982_b200 import sharding

    n_q, n_r = 4, 256
    n = n_q * n_r
    side = int(round(n_points ** 0.5))
    pts = eff.sweep_points(side, n_points // side)
    tgt = eff.sweep_target(n_r)
    a, b = sharding.shard_bounds(pts.shape[0], world, rank)
    mine = pts[a:b]
    state = {}

    def rebuild():  # fresh operators on the device (writes 16 GiB / world: L2 flushed)
        state["mats"], state["mx"] = npd.build_transmon_resonator_batch(mine, n_q, n_r, with_max_abs=True)

    def step():
        state["out"] = npd._run_batch_inplace(state["mats"], tgt, 1e-12, None, state["mx"])

    rebuild()
    step()
    tot = []
    lib.profile_read(reset=True)
    lib.profile_enable(True)
    for _ in range(2):
        rebuild()
        tot += time_steps(torch, step, 1, lambda: None, world)
    lib.profile_enable(False)
    prof = lib.profile_read(reset=True)
    applied = state["out"][0].cpu().numpy()
    conv = state["out"][1].cpu().numpy()
    rot_local = int(applied.sum())
    rot = int(round(sum_over_ranks(torch, rot_local, world)))
    all_conv = sum_over_ranks(torch, float(conv.all()), world) == world
    per = max_over_ranks(torch, sum(tot) / len(tot), world)
    # kernel time per sweep (the warp driver, then the shared-memory driver
    # for the tail: both record as npad_run_kernel)
    kms = max_over_ranks(torch, prof["npad_run_kernel"][0] / len(tot), world)
    ach = 96 * n * rot / world / (kms * 1e-3) / 1e9  # per GPU
    # e2e: host (omega_q, alpha, omega_r, g) rows in -> per-point applied,
    # converged and final diagonal on the host (rank 0 gathers), through the
    # public API (npad_sweep_transmon on 1 GPU, sharding.sweep_sharded on N)
    del state["mats"]

    def e2e_step():
        if world == 1:
            r = eff.npad_sweep_transmon(pts, n_q, n_r, tgt, tol=1e-12)
            state["e2e"] = (r.applied, r.converged, r.diagonals())
            del r
        else:
            r = sharding.sweep_sharded(pts, n_q, n_r, tgt, tol=1e-12)
            state["e2e"] = r.gather()
            del r

    e2e_step()  # warm-up (allocator, pinned buffers)
    e2e_ms = time_steps(torch, e2e_step, 2, lambda: None, world)
    e2e_per = max_over_ranks(torch, sum(e2e_ms) / len(e2e_ms), world)
    assert int(state["e2e"][0].sum()) == rot
    cpu = None
    if rank == 0:  # CPU: reference algorithm on 2 sweep points, first 60 rotations each
        t0 = time.perf_counter()
        crot = 0
        for row in pts[:2]:
            h = eff.transmon_resonator_hamiltonian(n_q, n_r, omega_q=row[0], alpha=row[1], omega_r=row[2],
                                                   g=row[3]).data
            crot += npad_oracle.run_full_scan(h, tgt, tol=1e-12, max_iter=60)["applied"]
        cpu = crot / (time.perf_counter() - t0)
    return {"workload": f"config 4: NPAD sweep {pts.shape[0]} (g, Delta) points, transmon4 x resonator256 (dim 1024),"
                        f" subspace target 10 levels, tol 1e-12, "
                        + ("one GPU" if world == 1 else f"points split over {world} GPUs"),
            "metric": "NPAD rotations/s", "unit": "rotations/s", "value": rot / (per * 1e-3), "rotations": rot,
            "n_gpus": world, "scaling": "strong", "all_converged": bool(all_conv), "ms_per_sweep": per,
            "e2e": {"value": rot / (e2e_per * 1e-3), "unit": "rotations/s", "ms_per_sweep": e2e_per,
                    "h2d_bytes_per_step": int(pts.nbytes),
                    "d2h_bytes_per_step": int(pts.shape[0] * (n * 8 + 8 + 1)),
                    "path": "npad_sweep_transmon(host points) / sharding.sweep_sharded(...).gather(): per-point "
                            "applied, converged, final diagonal to the host"},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peaks[0], "unit": "GB/s", "frac": ach / peaks[0],
                         "per": "GPU", "bytes_per_rotation": 96 * n,
                         "traffic": traffic_from_profiles("npad_trows_warp_kernel@sweep")},
            "cpu_baseline": {"value": cpu, "unit": "rotations/s", "cores": 1, "kind": "port",
                             "sample": "first 60 rotations of 2 sweep points, oracle run_full_scan"}}


def _magnus5_problem(eff, n_int=4096):
    L = 12
    ch = eff.heisenberg_chain_hamiltonians(L)
    full = eff.synthetic_transfer_pulse(25.0, 4096 * 8 + 1, seed=7)
    grid = eff.ControlGrid(0.0, 25.0 * n_int / 4096, full.signals[:, :n_int * 8 + 1])
    psi0 = np.zeros(1 << L, dtype=complex)
    psi0[0] = 1
    return ch, grid, psi0


def _herm_fraction(n, bm=128, bn=64):
    """Share of the 8 N^3 of a complex GEMM the Hermitian kernel computes (the
    128 x 64 tiles meeting the lower triangle)."""
    tm, tn = -(-n // bm), -(-n // bn)
    return sum(min(2 * r + 2, tn) for r in range(tm)) / (tm * tn)


def _dmma_sample(torch, eff, lib, ch, grid_full, psi0, n_int=32):
    """The DMMA engine on the first n_int intervals of config 5 (the FP64
    tensor-pipe roofline of the north star; the default engine is int8)."""
    from paper_2411_09982_b200 import magnus as mg

    old = lib.load().qch_set_herm_gemm(0)
    try:
        g = eff.ControlGrid(0.0, 25.0 * n_int / 4096, grid_full.signals[:, : n_int * 8 + 1])
        d_psi = lib.to_device(psi0)
        mg.evolve_device(ch, g, n_int, d_psi, check=False, order=2)  # warm-up (allocations)
        torch.cuda.synchronize()
        lib.profile_read(reset=True)
        lib.profile_enable(True)
        f0 = float(lib.load().qch_dmma_flops())
        ms = time_steps(torch, lambda: mg.evolve_device(ch, g, n_int, d_psi, check=False, order=2), 1, lambda: None,
                        1)[0]
        fl = float(lib.load().qch_dmma_flops()) - f0
        lib.profile_enable(False)
        prof = lib.profile_read(reset=True)
    finally:
        lib.load().qch_set_herm_gemm(old)
    g_ms = sum(v[0] for k, v in prof.items() if k.startswith("zgemm"))
    return {"intervals": n_int, "intervals_per_s": n_int / (ms * 1e-3), "gemm_ms": g_ms,
            "achieved_tflops": fl / (g_ms * 1e-3) / 1e12 if g_ms else None}


def sec_magnus4096(torch, eff, lib, args, fp64, world=1, rank=0, n_int=4096):
    """Config 5 at its stated size: Magnus order 2 on the 12-spin Heisenberg
    chain (dim 4096), ALL 4096 intervals.  One GPU: the public evolve()
    (host psi0 + signals in, host trajectory out), its device phase timed
    with CUDA events (value) and the whole call (e2e).  N GPUs: the relay
    (sharding.evolve_relay, chunks round-robin, psi passed rank to rank) +
    the trajectory gather to the host.  The Hermitian products run on the
    int8 tensor cores (Ozaki slices, tcgen05) — the default engine; a
    32-interval sample on the DMMA engine is reported beside it."""
    from oracle import expm_oracle
    from paper_2411_09982_b200 import magnus as mg
    from paper_2411_09982_b200 import sharding

    ch, grid, psi0 = _magnus5_problem(eff, n_int)
    n = ch.dim
    ch.device_operators()
    # warm-up: 2 intervals (allocations, attributes, commutators)
    g2 = eff.ControlGrid(0.0, 25.0 * 2 / 4096, grid.signals[:, :17])
    if world == 1:
        eff.evolve(ch, g2, 2, psi0, order=2, check=False)
    else:
        sharding.evolve_relay(ch, eff.ControlGrid(0.0, 25.0 * world / 4096, grid.signals[:, :8 * world + 1]), world,
                              psi0, order=2, check=False, chunk=1)
    torch.cuda.synchronize()
    lib.profile_read(reset=True)
    lib.profile_enable(True)
    fl0 = float(lib.load().qch_dmma_flops())
    op0 = float(lib.load().qch_int8_ops())
    eq0 = float(lib.load().qch_int8_fp64_equiv_flops())
    if world == 1:
        mg.PHASE_TIMING = True
        ms = time_steps(torch, lambda: eff.evolve(ch, grid, n_int, psi0, order=2, check=False), 1, lambda: None, 1)
        mg.PHASE_TIMING = False
        ph = dict(mg.LAST_PHASES)
        dev_ms, e2e_ms = ph["device_ms"], ms[0]
        d2h = (n_int + 1) * n * 16
    else:
        res = {}

        def relay():
            res["r"] = sharding.evolve_relay(ch, grid, n_int, psi0, order=2, check=False)

        def gather():
            tr = res["r"].gather()
            if rank == 0:
                res["host"] = lib.to_host(tr)

        dev_ms = max_over_ranks(torch, time_steps(torch, relay, 1, lambda: None, world)[0], world)
        g_ms = max_over_ranks(torch, time_steps(torch, gather, 1, lambda: None, world)[0], world)
        e2e_ms = dev_ms + g_ms
        d2h = (n_int + 1) * n * 16
    lib.profile_enable(False)
    prof = lib.profile_read(reset=True)
    engine = int(lib.load().qch_set_herm_gemm(-1))
    fl_ref = 17 * 8 * n**3
    # the dominant kernel of the default engine: oz_gemm (int8 tensor cores)
    oz_ms = max_over_ranks(torch, prof.get("oz_gemm", (0.0, 0))[0], world)
    ops = sum_over_ranks(torch, float(lib.load().qch_int8_ops()) - op0, world)
    eqf = sum_over_ranks(torch, float(lib.load().qch_int8_fp64_equiv_flops()) - eq0, world)
    dm_ms = max_over_ranks(torch, sum(v[0] for k, v in prof.items() if k.startswith("zgemm")), world)
    dm_fl = sum_over_ranks(torch, float(lib.load().qch_dmma_flops()) - fl0, world)
    mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    if fp64.get("cublaslt_int8_tops"):
        i8_peak, i8_kind = fp64["cublaslt_int8_tops"], "measured live: cuBLASLt int8 GEMM 8192^3 (torch._int_mm), best of 5"
    else:
        i8_peak = 2.0 * mp.get("bf16_tflops", 1590.0)
        i8_kind = "dense int8 = 2 x the measured cuBLAS bf16 burst of MEASURED_PEAKS.json (nominal 4500)"
    kernels_ms = {k: v[0] for k, v in prof.items()}
    if engine == 1 and oz_ms:
        ach = ops / world / (oz_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": "oz_gemmw_kernel<256, pair> (tcgen05.mma.cta_group::2 kind::i8, 256 x 256 CTA-pair tiles, TMEM, TMA; Ozaki slices)",
                "achieved": ach, "peak": i8_peak, "unit": "TOPS (int8)", "frac": ach / i8_peak,
                "peak_kind": i8_kind, "nominal_peak": 4500.0,
                "ops_basis": "int8 tensor ops issued by the library (qch_int8_ops): 3 real products per complex "
                             "product x the slice pairs each product uses (adaptive plan: 36 / 28 / 21 / 15 for "
                             "8 / 7 / 6 / 5 slices) x 2 M N K per computed tile",
                "gemm_ms": oz_ms,
                "fp64_equivalent_tflops": eqf / world / (oz_ms * 1e-3) / 1e12,
                "fp64_equivalent_note": "complex-product flops the int8 GEMMs stand in for (8 M N K over the computed "
                                        "tiles, qch_int8_fp64_equiv_flops) / int8 GEMM time -- vs the live DMMA peak "
                                        f"{fp64.get('dmma', 0):.1f} TFLOP/s",
                "kernel_ms": kernels_ms,
                "traffic": traffic_from_profiles("oz_gemmw_kernel@oz")}
    else:
        ach = dm_fl / world / (dm_ms * 1e-3) / 1e12 if dm_ms else None
        roof = {"bound": "tensor", "kernel": "zgemm_tma_kernel (DMMA, TMA-fed)", "achieved": ach,
                "peak": fp64.get("dmma"), "unit": "TFLOP/s",
                "frac": (ach / fp64["dmma"]) if ach and fp64.get("dmma") else None,
                "gemm_ms": dm_ms, "kernel_ms": kernels_ms}
    roof["reference_equivalent_tflops"] = fl_ref * n_int / (dev_ms * 1e-3) / 1e12
    roof["flops_per_interval_reference"] = fl_ref
    dmma = None
    if world == 1 and rank == 0:
        dmma = _dmma_sample(torch, eff, lib, ch, grid, psi0)
        if dmma.get("achieved_tflops") and fp64.get("dmma"):
            dmma["frac_of_dmma_peak"] = dmma["achieved_tflops"] / fp64["dmma"]
    cpu = None
    if rank == 0:  # the reference's _expm_minus_i (18-term Taylor, expm.py:56-71) on ONE interval, host cores
        try:
            from threadpoolctl import threadpool_info

            blas = [(i.get("internal_api"), i.get("num_threads")) for i in threadpool_info()]
        except Exception:  # pragma: no cover
            blas = None
        hb = ch.drift.to_dense() * (25.0 / 4096)
        t0 = time.perf_counter()
        expm_oracle.expm_minus_i(hb)
        cpu_s = time.perf_counter() - t0
        cpu = {"value": 1.0 / cpu_s, "unit": "intervals/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"one interval's propagator at N = 4096 (oracle expm_minus_i = the reference's 18-term "
                         f"Taylor, 17 complex GEMMs on numpy/OpenBLAS), {cpu_s:.1f} s; BLAS threads {blas}"}
    return {"workload": f"config 5: Magnus 12-spin Heisenberg chain (dim 4096), order 2, ALL {n_int} intervals, "
                        + ("one GPU" if world == 1 else f"relay over {world} GPUs"),
            "metric": "Magnus intervals/s", "unit": "intervals/s", "value": n_int / (dev_ms * 1e-3),
            "intervals": n_int, "n_gpus": world, "scaling": "strong", "ms_per_evolve": dev_ms,
            "engine": "int8 tensor cores (Ozaki, tcgen05)" if engine == 1 else "DMMA",
            "e2e": {"value": n_int / (e2e_ms * 1e-3), "unit": "intervals/s", "ms": e2e_ms,
                    "h2d_bytes_per_step": int(grid.signals.nbytes + psi0.nbytes), "d2h_bytes_per_step": int(d2h),
                    "path": "evolve(host psi0, host grid) -> host trajectory" if world == 1
                            else "sharding.evolve_relay + gather -> host trajectory on rank 0"},
            "roofline": roof,
            "dmma_engine_sample": dmma,
            "cpu_baseline": cpu}


def sec_midsize(torch, eff, lib, args, fp64, L=8, n_int=2048):
    """dense propagation at mid-size N (8-spin Heisenberg
    chain, N = 256) with the reference's default check=True."""
    from oracle import magnus_oracle
    from paper_2411_09982_b200 import magnus as mg

    n = 1 << L
    ch = eff.heisenberg_chain_hamiltonians(L)
    pulse = eff.synthetic_transfer_pulse(25.0, n_int * 8 + 1, seed=7)
    grid = eff.ControlGrid(0.0, 25.0, pulse.signals)
    psi0 = np.zeros(n, dtype=complex)
    psi0[0] = 1
    d_psi = lib.to_device(psi0)
    ch.device_operators()

    def step():
        mg.evolve_device(ch, grid, n_int, d_psi, check=True, order=2)

    step()
    lib.profile_read(reset=True)
    lib.profile_enable(True)
    fl0 = float(lib.load().qch_dmma_flops())
    ms = time_steps(torch, step, 3, lambda: None, 1)
    fl = (float(lib.load().qch_dmma_flops()) - fl0) / 3  # executed DMMA flops per step (library count)
    lib.profile_enable(False)
    prof = lib.profile_read(reset=True)
    per = sum(ms) / len(ms)
    g_ms = sum(v[0] for k, v in prof.items() if k.startswith("zgemm")) / 3
    rp = int(lib.load().qch_zgemm_real_products())
    frac_h = _herm_fraction(n)
    ach = fl / (g_ms * 1e-3) / 1e12 if g_ms else None
    chain_ms = sum(v[0] for k, v in prof.items() if k.startswith("chain_")) / 3
    # CPU: the oracle (numpy restatement of evolve, 18-term Taylor, order 2) on 8 intervals
    k_cpu = 8
    d0 = ch.drift.to_dense()
    ctr = np.stack([c.to_dense() for c in ch.controls])
    sub_sig = grid.signals[:, : k_cpu * 8 + 1]
    t0 = time.perf_counter()
    magnus_oracle.evolve(d0, ctr, sub_sig, 0.0, 25.0 * k_cpu / n_int, k_cpu, psi0, order=2)
    cpu = k_cpu / (time.perf_counter() - t0)
    return {"workload": f"SURVEY 8(f) rank 2: Magnus, {L}-spin Heisenberg chain (dim {n}), {n_int} intervals, "
                        f"order 2, check=True",
            "metric": "Magnus intervals/s", "unit": "intervals/s", "value": n_int / (per * 1e-3),
            "ms_per_step": per, "gemm_ms": g_ms, "chain_ms": chain_ms,
            "roofline": {"bound": "tensor", "kernel": "zgemm_tma_kernel (DMMA, TMA-fed)", "achieved": ach, "peak": fp64.get("dmma"),
                         "unit": "TFLOP/s", "frac": (ach / fp64["dmma"]) if ach and fp64.get("dmma") else None,
                         "flops_basis": f"executed DMMA flops ({2 * rp} N^3 per complex GEMM, the computed "
                                        f"share {frac_h:.3f} for Hermitian half-GEMMs)"},
            "cpu_baseline": {"value": cpu, "unit": "intervals/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": f"{k_cpu} intervals, oracle/magnus_oracle.evolve (numpy/OpenBLAS)"}}


def sec_givens(torch, eff, lib, args, peaks, sizes=(10**5, 10**6, 10**7, 10**8)):
    """SURVEY 8(f) rank 1 / the paper's Fig. 4 protocol (bench_givens,
    experiments.py:420-453): ONE Givens rotation eliminating the smallest
    coupling (0, 1) of the sparse ladder a^dag a + (a + a^dag) (CSR, built on
    the device), through the public eliminate_coupling."""
    from oracle import npad_oracle

    rows = []
    for n in sizes:
        op = eff.ladder_test_hamiltonian_device(n)
        st0 = eff.NPADState.from_operator(op)
        for _ in range(2):
            eff.eliminate_coupling(st0, 0, 1)
        torch.cuda.synchronize()
        lib.profile_read(reset=True)
        lib.profile_enable(True)
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            out = eff.eliminate_coupling(st0, 0, 1)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / reps
        lib.profile_enable(False)
        prof = lib.profile_read(reset=True)
        nnz = 3 * n - 3
        # algorithmic bytes: the input CSR read and the new CSR written
        # (int64 indptr, int32 indices, complex128 values)
        byts = 2 * (8 * (n + 1) + 20 * nnz)
        k = prof.get("npad_sparse_rotate")
        kms = k[0] / k[1] if k else None
        s_ms = prof["npad_sparse_stream"][0] / prof["npad_sparse_stream"][1] if "npad_sparse_stream" in prof else None
        row = {"n": n, "nnz_in": nnz, "nnz_out": out.current.nnz, "ms_per_rotation_e2e": wall * 1e3,
               "ms_kernels": kms, "ms_streaming_passes": s_ms,
               "achieved_gbs_streaming": byts / (s_ms * 1e-3) / 1e9 if s_ms else None}
        if n <= 10**6:
            host = eff.ladder_test_hamiltonian(n).data
            t0 = time.perf_counter()
            npad_oracle.eliminate_sparse(host, 0, 1)
            row["cpu_ms"] = (time.perf_counter() - t0) * 1e3
        rows.append(row)
        del op, st0, out
    big = rows[-1]
    return {"workload": "SURVEY 8(f) rank 1 — bench_givens (PAPER.md:180-183): one sparse Givens rotation on the "
                        "ladder a^dag a + (a + a^dag), N = 1e5..1e8 (CSR on the device)",
            "metric": "rotation time", "unit": "ms", "value": big["ms_per_rotation_e2e"], "higher_is_better": False,
            "sizes": rows,
            "roofline": {"bound": "hbm", "achieved": big["achieved_gbs_streaming"], "peak": peaks[0], "unit": "GB/s",
                         "frac": (big["achieved_gbs_streaming"] / peaks[0]) if big["achieved_gbs_streaming"] else None,
                         "note": "the two streaming passes (new indptr, shifted copy of every other row) of the "
                                 "largest size; algorithmic bytes = input CSR read + output CSR write"},
            "cpu_baseline": {"value": rows[1].get("cpu_ms"), "unit": "ms at N = 1e6", "cores": 1, "kind": "port",
                             "sample": "oracle/npad_oracle.eliminate_sparse (scipy restatement of "
                                       "_conjugate_sparse) at N = 1e5 and 1e6"}}


# --------------------------------------------------------------- reference --

def run_reference(args, world, rank):
    """--impl reference: the reference's CPU algorithm (oracle port of
    effham.magnus.evolve + the 2nd-order restatement) on the host cores, the
    headline config's metric, bounded sample per step; rank 0 only."""
    if rank != 0:
        return
    from concurrent.futures import ProcessPoolExecutor

    from paper_2411_09982_b200 import models as eff_models

    cores = os.cpu_count() or 1
    chunk = 20000
    per_step = chunk * cores
    ex = ProcessPoolExecutor(max_workers=cores)
    list(ex.map(_ref_chunk, [200] * cores))  # spawn + import outside the timing

    def one_step():
        t0 = time.perf_counter()
        list(ex.map(_ref_chunk, [chunk] * cores))
        return time.perf_counter() - t0

    for _ in range(max(1, args.warmup)):
        one_step()
    ts = [one_step() for _ in range(args.steps)]
    ex.shutdown()
    per = sum(ts) / len(ts)
    value = per_step / per
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "intervals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic",
            "config": {"workload": "config 2: Magnus driven 3-level transmon, order 2, 1e5 intervals "
                                   "(CPU: bounded sample per step)", "order": 2, "dim": 3, "sub": SUB},
            "cpu_baseline": {"value": value, "unit": "intervals/s", "cores": cores, "kind": "port",
                             "sample": f"{cores} processes x {chunk} intervals per step (oracle/magnus_oracle.evolve,"
                                       f" numpy restatement of effham.magnus.evolve + 2nd-order term)"},
            "e2e": {"value": value, "unit": "intervals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _ref_chunk(n_int):
    sys.path.insert(0, str(ROOT))
    from paper_2411_09982_b200 import models as eff_models

    return cpu_magnus_sample(eff_models, n_int)[0]


# -------------------------------------------------------------------- main --

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--secondary", default="all")
    ap.add_argument("--npad4096-rotations", type=int, default=0, help="0 = run to convergence")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch

    # QCH_BENCH_BACKEND=gloo + QCH_BENCH_SAME_GPU=1: dry-run the multi-rank
    # paths with every rank on GPU 0 (functional check only, not a timing)
    backend = os.environ.get("QCH_BENCH_BACKEND", "nccl")
    dev = 0 if os.environ.get("QCH_BENCH_SAME_GPU") == "1" else local
    torch.cuda.set_device(dev)
    local = dev
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import _lib as lib

    lib.load(build_if_missing=False)
    hbm_peak, hbm_src = measured_peaks()
    fp64 = fp64_peaks(torch, lib)
    head = run_headline(torch, eff, lib, args, world, rank, local)

    secondary = []
    if args.secondary != "none":
        want = {"npad60", "npad4096", "sweep", "magnus4096", "givens", "midsize"} if args.secondary == "all" else set(
            args.secondary.split(","))
        peaks = (hbm_peak, hbm_src)
        single = rank == 0 and world == 1  # replicas-only paths: one GPU
        if single and "npad60" in want:
            secondary.append(sec_npad60(torch, eff, lib, args, peaks))
        if single and "npad4096" in want:
            secondary.append(sec_npad4096(torch, eff, lib, args, peaks, args.npad4096_rotations or None))
        if "sweep" in want:  # sharded over the ranks when N > 1
            secondary.append(sec_sweep(torch, eff, lib, args, peaks, world, rank))
        if "magnus4096" in want:  # relay over the ranks when N > 1
            secondary.append(sec_magnus4096(torch, eff, lib, args, fp64, world, rank))
        if single and "givens" in want:
            secondary.append(sec_givens(torch, eff, lib, args, peaks))
        if single and "midsize" in want:
            secondary.append(sec_midsize(torch, eff, lib, args, fp64))

    if rank == 0:
        cpu_v, cpu_t = cpu_magnus_sample(__import__("paper_2411_09982_b200.models", fromlist=["x"]), 60000)
        roof = head["roof"]
        achieved = roof["flops_per_launch"] / (roof["launch_ms"] * 1e-3) / 1e12 if roof else None
        line = {
            "metric": METRIC,
            "value": head["value"],
            "unit": "intervals/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": head["per_step"],
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64 (complex128)",
            "data": "synthetic (driven transmon, SURVEY.md §8(d) config 2)",
            "config": {"workload": "config 2: Magnus time coarse-graining, driven 3-level transmon, 1e5 intervals per "
                                   "GPU, 2nd order, sub=4 samples/interval, check=False (as experiments.py:369)",
                       "intervals_total": head["m"], "order": 2, "dim": 3, "controls": 2,
                       "parallelism": f"interval-sharded x{world}" if world > 1 else "single GPU",
                       "l2": "flushed between timed steps (256 MiB write, outside the events)"},
            "e2e": {"value": head["e2e"][0], "unit": "intervals/s", "h2d_bytes_per_step": head["e2e"][1],
                    "d2h_bytes_per_step": head["e2e"][2], "signals": "page-locked host array",
                    "pageable_value": head["e2e_pageable"],
                    "pageable_note": "same call with the plain pageable numpy signals a reference caller passes"},
            "gpu_launches": head["launches"],
            "clocks": head["clocks"],
            "roofline": {"bound": "fp64", "kernel": "magnus_fused_kernel", "achieved": achieved,
                         "peak": fp64["dfma"], "unit": "TFLOP/s",
                         "frac": (achieved / fp64["dfma"]) if achieved else None,
                         "traffic": traffic_from_profiles("magnus_fused_kernel@magnus2"),
                         "peak_kind": "FP64 FMA pipe, measured live by bench.py (DFMA probe); MEASURED_PEAKS.json "
                                      "has no FP64 entry. Per-interval 3x3 expm is FP64-FMA work, not tensor work",
                         "flops_basis": "SURVEY.md 8(d) per-interval figure of the reference algorithm (18-term "
                                        "Taylor); the kernel evaluates the same series to 2^-56 with fewer flops "
                                        "(executed_* keys)",
                         "executed_achieved": (roof["executed_flops_per_launch"] / (roof["launch_ms"] * 1e-3) / 1e12)
                         if roof else None,
                         "flops_per_launch": roof["flops_per_launch"] if roof else None,
                         "kernel_share_of_step": roof["kernel_share_of_step"] if roof else None},
            "cpu_baseline": {"value": cpu_v, "unit": "intervals/s", "cores": 1, "kind": "port",
                             "sample": f"60000 intervals of the same configuration ({cpu_t:.1f} s), "
                                       "oracle/magnus_oracle.evolve order 2"},
            "fp64_peaks_tflops": fp64,
            "hbm_peak": {"gbs": hbm_peak, "source": hbm_src},
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
