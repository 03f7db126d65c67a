#!/usr/bin/env python3
"""RN-AMG setup + solve benchmark (BASELINE.json metric) on B200.

Workload (default --config 5, the largest BASELINE config: 37.8 M nonzeros): 2D plane-
strain linear elasticity, bilinear Q1 on a 1024 x 1024 element grid, 2 DOFs per node
(2,099,200 DOFs), E = 1, nu = 0.3, left edge clamped; near-nullspace B = 3 rigid-body
modes; node-wise block SOC theta = 0.1, 2x2-block aggregation, 4 energy-min CG
iterations with the 3-column constraint projection, V(1,1) weighted Jacobi, PCG to
1e-8 relative residual.  Synthetic input from the config generator (b seeded, seed 3).
--config 1..4 selects the other BASELINE configs.

One step = rn_setup + solve of that problem.  `value` is the device time of a step
with A, B and b already resident in HBM (CUDA events on the library stream, L2
flushed before every step); `e2e` is the same step through the public C ABI with
pinned host buffers (host->device copies of A, B, b and the device->host read of x
inside the timed region).  Every global sum is the reference's left-to-right chain
bit for bit (the default context mode), so the hierarchy, the iteration count and the
residual history are the reference's.

--impl reference times the reference's own CPU implementation of the path
(oracle/_ref: the reference headers compiled unmodified against the Eigen stand-in)
on the box's host, on inputs from oracle/build/libconfiggen.so (libamgcu.so is not
loaded).  One reference setup+solve at full size takes minutes (its injection scans
every node per aggregate), so each step is a bounded sample -- the same config on a
smaller grid -- and `value` scales the sample's seconds by the DOFs ratio (a lower
bound on the reference's full-size time).  The GPU arm's cpu_baseline samples the
own-code restatement (oracle/rnamg_port.cpp) the same way.

Multi-GPU (--gpus N under torchrun): replicas only -- every rank solves its
own copy of the problem, no data-path collective;
torch.distributed is used for the barrier and the max-over-ranks timing.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "RN-AMG setup+solve s to 1e-8 rel resid; achieved HBM GB/s vs peak"
CONFIG_NAMES = {1: "C1 2D Poisson 5-pt 256^2", 2: "C2 rotated anisotropic Q1 1024^2 elements (eps 1e-3, pi/8)",
                3: "C3 recirculating convection-diffusion 2048^2", 4: "C4 upwind transport 2048^2",
                5: "C5 Q1 plane-strain elasticity 1024^2 elements"}
DEFAULT_SIZE = {1: 256, 2: 1024, 3: 2048, 4: 2048, 5: 1024}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--size", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--family-timing", type=int, default=1,
                    help="1: CUDA events around the dominant kernel family's launches in the timed region")
    ap.add_argument("--max-restarts", type=int, default=50)
    ap.add_argument("--cpu-budget", type=float, default=float(os.environ.get("AMG_CPU_BUDGET_S", "200")),
                    help="seconds of CPU work the reference arm / cpu_baseline sample may take")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# kernel family -> kernel symbol captured by tools/ncu_capture.sh
PROFILE_TAG = "r04"  # profiles/<tag>_traffic.json, written by tools/ncu_summary.py
FAMILY_KERNEL = {"gauss_seidel_wavefront": "k_gs_seg_warp<3, 1>", "aggregate_lfmis": "k_lfmis_lists",
                 "spgemm": "k_spgemm_bitmap", "arnoldi_blas1": "k_seqsum<TAxpyDot, 16>", "blas1": "k_seqsum<TDot, 16>",
                 "emin_masked_product": "k_masked_band<3, 0>", "vcycle_relax0_residual": "k_relax0_residual",
                 "vcycle_post_relax": "k_jacobi_sweep", "vcycle_prolong": "k_prolong", "krylov_spmv": "k_sell_spmv",
                 "vcycle_coarse_fused": "k_vcycle_fused", "coarse_solve": "k_gauss_jordan", "emin_cg": "k_cg_columns"}


def ncu_traffic(family):
    """DRAM bytes (read + write) of the family's largest captured launch, from the committed
    ncu --set full summary (profiles/<PROFILE_TAG>_traffic.json, written by tools/ncu_summary.py)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", f"{PROFILE_TAG}_traffic.json")
    kern = FAMILY_KERNEL.get(family)
    try:
        launches = json.load(open(path)).get(kern, [])
    except (OSError, ValueError):
        return None, "no ncu capture"
    if not launches:
        return None, "no ncu capture"
    top = max(launches, key=lambda d: d["dram_bytes"])
    return top["dram_bytes"], f"ncu --set full, {kern} grid {top['grid']} (profiles/{PROFILE_TAG}_ncu_summary_table.md)"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.rows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = sorted(float(r[0]) for r in rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def oracle_run(kind, config, size, max_restarts):
    """CPU run of one setup + solve (kind 'port' or 'ref') on inputs from the oracle-side
    generator library (no libamgcu.so); returns (setup_s, solve_s, iterations, converged, levels)."""
    from oracle.pyoracle import Oracle, config_options, generate_config
    A, B, Bh, b = generate_config(config, size)
    so, vo = config_options(config)
    o = Oracle(kind)
    t0 = time.perf_counter()
    h = o.setup(A, B, so, Bh)
    t1 = time.perf_counter()
    x, rep = o.solve(h, b, None, vo)
    its = rep.iterations
    restarts = 0
    while vo.method == 2 and not rep.converged and not rep.diverged and restarts < max_restarts:
        x, rep = o.solve(h, b, x, vo)
        its += rep.iterations
        restarts += 1
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, its, bool(rep.converged), h.n_levels()


def dofs(config, size):
    """unknowns of config `config` at grid size `size` (problems.cpp)"""
    if config == 1:
        return size * size
    if config == 2:
        return (size - 1) * (size - 1)
    if config == 5:
        return 2 * size * (size + 1)
    return size * size


SAMPLE_SIZES = {1: (256, 192, 128, 96), 2: (512, 384, 256, 128), 3: (512, 384, 256, 128),
                4: (512, 384, 256, 128), 5: (512, 384, 256, 128)}


def cpu_sample(kind, config, size, runs, budget_s, max_restarts):
    """Bounded CPU sample of the workload: the same config on a smaller grid, sized so
    `runs` setup+solves fit in budget_s.  A calibration run at the smallest candidate
    grid (untimed; it also loads the library) predicts the others with a super-linear
    model (t ~ n^1.7, the reference's measured C5 growth from 256^2 to 512^2).
    Returns (sample_size, calibration_s)."""
    cands = [s for s in SAMPLE_SIZES[config] if s <= size] or [size]
    base = cands[-1]
    r = oracle_run(kind, config, base, max_restarts)
    t_base = r[0] + r[1]
    for s in cands:
        est = t_base * (dofs(config, s) / dofs(config, base)) ** 1.7
        if runs * est <= budget_s or s == base:
            return s, t_base
    return base, t_base


def scaled_value(t_sample, config, size, sample):
    """seconds of the full workload from a sample: t x (DOFs ratio) -- linear scaling, a
    lower bound for the reference (its injection scan grows with n_agg x n)"""
    return t_sample * dofs(config, size) / dofs(config, sample)


def config_dict(config, size, n, nnz):
    """the workload description both arms print (identical dicts)"""
    return {"workload": CONFIG_NAMES[config], "config": config, "size": size, "n": n, "nnz": nnz,
            "l2": "GPU arm: flushed (256 MB write) before every step"}


def run_reference(args, ws, rank):
    """--impl reference: the reference's CPU implementation (oracle/_ref: the reference
    headers compiled unmodified), rank 0 only, inputs from oracle/build/libconfiggen.so."""
    if rank != 0:
        return
    from oracle.pyoracle import available
    config = args.config
    size = args.size or DEFAULT_SIZE[config]
    if not available("ref"):
        kind = "port"
        why = "oracle/_ref not built; own-code restatement (rnamg_port.cpp) timed instead"
    else:
        kind = "ref"
        why = None
    from oracle.pyoracle import generate_config
    A_full = generate_config(config, size)[0]  # the workload's shape, for the config dict
    n_full, nnz_full = A_full.n_rows, A_full.nnz()
    del A_full
    t0 = time.perf_counter()
    runs = args.warmup + max(1, args.steps)
    sample, t_cal = cpu_sample(kind, config, size, runs, args.cpu_budget, args.max_restarts)
    for _ in range(args.warmup):
        oracle_run(kind, config, sample, args.max_restarts)
    timed = [oracle_run(kind, config, sample, args.max_restarts) for _ in range(max(1, args.steps))]
    wall = time.perf_counter() - t0
    per_step = [r[0] + r[1] for r in timed]
    t_s = sum(per_step) / len(per_step)
    v = scaled_value(t_s, config, size, sample)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (config generator, seeded)",
        "config": config_dict(config, size, n_full, nnz_full),
        "result": {"sample_size": sample, "sample_s": t_s,
                   "setup_s": sum(r[0] for r in timed) / len(timed), "solve_s": sum(r[1] for r in timed) / len(timed),
                   "iterations": timed[0][2], "converged": timed[0][3], "levels": timed[0][4]},
        "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "reference" if kind == "ref" else "port",
                         "sample": f"config {config} at {sample}^2 ({dofs(config, sample)} DOFs), one setup+solve "
                                   f"per step, single thread (the reference is single-threaded); value = sample "
                                   f"seconds x DOFs ratio {dofs(config, size) / dofs(config, sample):.3f} (linear "
                                   f"scaling: a lower bound, the reference's injection scan grows as n_agg x n); "
                                   f"{args.warmup} warm-ups + {len(timed)} timed steps at the sample size, "
                                   f"calibration {t_cal:.1f}s, wall {wall:.1f}s",
                         "host_cores": os.cpu_count()},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if why:
        line["note"] = why
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import numpy as np
    import torch

    import paper_1610_03154_b200.api as api
    from paper_1610_03154_b200._abi import CsrC, SolveReportC, f64p
    lib = api.lib

    # replicas only: the barrier and the max-over-ranks come from the
    # package's replicas helpers, the same code the world-size-2 gloo test exercises
    import paper_1610_03154_b200.replicas as replicas
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    dist = replicas.init("nccl")
    config = args.config
    size = args.size or DEFAULT_SIZE[config]
    A, B, Bh, b = api.generate_config(config, size)
    so, vo = api.config_options(config)
    n, nnz, k = A.n_rows, A.nnz(), B.k
    ctx = api.Context(local)

    # device-resident inputs
    d_rp = torch.from_numpy(A.row_offsets).to(device)
    d_ci = torch.from_numpy(A.col_indices).to(device)
    d_va = torch.from_numpy(A.values).to(device)
    d_B = torch.from_numpy(B.data).to(device)
    d_Bh = torch.from_numpy(Bh.data).to(device) if Bh is not None else None
    d_b = torch.from_numpy(b).to(device)
    d_x = torch.zeros(n, dtype=torch.float64, device=device)
    dcsr = CsrC(n, A.n_cols, nnz, A.block_size, C.cast(d_rp.data_ptr(), C.POINTER(C.c_int32)),
                C.cast(d_ci.data_ptr(), C.POINTER(C.c_int32)), C.cast(d_va.data_ptr(), C.POINTER(C.c_double)))
    # pinned host copies for the e2e leg
    p_rp = torch.from_numpy(A.row_offsets).pin_memory()
    p_ci = torch.from_numpy(A.col_indices).pin_memory()
    p_va = torch.from_numpy(A.values).pin_memory()
    p_B = torch.from_numpy(B.data).pin_memory()
    p_Bh = torch.from_numpy(Bh.data).pin_memory() if Bh is not None else None
    p_b = torch.from_numpy(b).pin_memory()
    p_x = torch.zeros(n, dtype=torch.float64).pin_memory()
    hcsr = CsrC(n, A.n_cols, nnz, A.block_size, C.cast(p_rp.data_ptr(), C.POINTER(C.c_int32)),
                C.cast(p_ci.data_ptr(), C.POINTER(C.c_int32)), C.cast(p_va.data_ptr(), C.POINTER(C.c_double)))
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)  # 256 MB > 126 MB L2
    so_c = so.to_c()
    vo_c = vo.to_c()
    hist = np.zeros(4096)

    def solve_loop(h, bptr, xptr, device_side):
        rep = SolveReportC()
        its, conv = 0, False
        for r in range(args.max_restarts + 1):
            if device_side:
                ctx._chk(lib.amgcu_solve_device(h, bptr, xptr, C.byref(vo_c), C.byref(rep),
                                                hist.ctypes.data_as(f64p), 4096))
            else:
                ctx._chk(lib.amgcu_solve(h, C.cast(bptr, f64p), C.cast(xptr, f64p), C.byref(vo_c), C.byref(rep),
                                         hist.ctypes.data_as(f64p), 4096))
            its += rep.iterations
            conv = bool(rep.converged)
            if vo.method != 2 or conv or rep.diverged:  # GMRES(m): restart with the current x
                break
        return its, conv, rep

    def step_device():
        d_x.zero_()
        h = C.c_void_p()
        ctx._chk(lib.amgcu_ctx_timer_start(ctx.handle))
        ctx._chk(lib.amgcu_setup_device(ctx.handle, C.byref(dcsr), k, C.c_void_p(d_B.data_ptr()),
                                        C.c_void_p(d_Bh.data_ptr()) if d_Bh is not None else None, C.byref(so_c),
                                        C.byref(h)))
        its, conv, rep = solve_loop(h.value, C.c_void_p(d_b.data_ptr()), C.c_void_p(d_x.data_ptr()), True)
        ms = C.c_double()
        ctx._chk(lib.amgcu_ctx_timer_stop(ctx.handle, C.byref(ms)))
        nl, st = C.c_int32(), C.c_int32()
        lib.amgcu_hier_levels(h.value, C.byref(nl), C.byref(st))
        lib.amgcu_hier_destroy(h.value)
        return ms.value, its, conv, nl.value

    def step_e2e():
        p_x.zero_()
        h = C.c_void_p()
        ctx._chk(lib.amgcu_ctx_timer_start(ctx.handle))
        ctx._chk(lib.amgcu_setup(ctx.handle, C.byref(hcsr), k, C.cast(p_B.data_ptr(), f64p),
                                 C.cast(p_Bh.data_ptr(), f64p) if p_Bh is not None else None, C.byref(so_c),
                                 C.byref(h)))
        its, conv, rep = solve_loop(h.value, p_b.data_ptr(), p_x.data_ptr(), False)
        ms = C.c_double()
        ctx._chk(lib.amgcu_ctx_timer_stop(ctx.handle, C.byref(ms)))
        lib.amgcu_hier_destroy(h.value)
        return ms.value, its, conv

    def flush_l2():
        flush.fill_(1.0)
        torch.cuda.synchronize()

    # warm-up (also profiles every kernel family once to pick the dominant one)
    lib.amgcu_ctx_set_profiling(ctx.handle, 1)
    lib.amgcu_ctx_profile_reset(ctx.handle)
    for _ in range(args.warmup):
        flush_l2()
        step_device()
    fam_count = lib.amgcu_profile_family_count()
    lib.amgcu_profile_family_name.restype = C.c_char_p
    fams = []
    for f in range(fam_count):
        l_, ms_, by_ = C.c_int64(), C.c_double(), C.c_double()
        lib.amgcu_ctx_profile_query(ctx.handle, f, C.byref(l_), C.byref(ms_), C.byref(by_))
        fams.append((ms_.value, f, lib.amgcu_profile_family_name(f).decode(), l_.value, by_.value))
    fams.sort(reverse=True)
    lib.amgcu_ctx_profile_reset(ctx.handle)
    # time only the dominant kernel family inside the timed region (2 events per launch);
    # "other" (untagged launches) and families without an algorithmic byte model are not kernels to roof
    kernel_fams = [f for f in fams if f[4] > 0 and f[2] != "other"]
    lib.amgcu_ctx_set_profile_mask(ctx.handle, C.c_uint32(1 << kernel_fams[0][1]))
    if not args.family_timing:
        lib.amgcu_ctx_set_profiling(ctx.handle, 0)

    # timed region: device-resident inputs
    sampler = ClockSampler(local)
    replicas.barrier(dist)
    torch.cuda.synchronize()
    sampler.start()
    launches0 = ctx.launch_count()
    step_ms, its, conv, levels = [], 0, False, 0
    for _ in range(args.steps):
        flush_l2()
        ms, its, conv, levels = step_device()
        step_ms.append(ms)
    launches = (ctx.launch_count() - launches0) / max(1, args.steps)
    torch.cuda.synchronize()
    replicas.barrier(dist)
    clocks = sampler.stop()
    fam_stats = {}
    for f in range(fam_count):
        l_, ms_, by_ = C.c_int64(), C.c_double(), C.c_double()
        lib.amgcu_ctx_profile_query(ctx.handle, f, C.byref(l_), C.byref(ms_), C.byref(by_))
        if l_.value:
            fam_stats[lib.amgcu_profile_family_name(f).decode()] = {
                "launches": l_.value, "ms": ms_.value, "algorithmic_bytes": by_.value}
    lib.amgcu_ctx_set_profiling(ctx.handle, 0)
    mean_ms = replicas.max_over_ranks(sum(step_ms) / len(step_ms), dist, device)

    # e2e: the public C ABI with pinned host buffers
    e2e_ms = []
    for _ in range(max(1, args.steps)):
        flush_l2()
        ms, _, _ = step_e2e()
        e2e_ms.append(ms)
    e2e_mean = replicas.max_over_ranks(sum(e2e_ms) / len(e2e_ms), dist, device)
    h2d = 4 * (n + 1) + 12 * nnz + 8 * n * k * (2 if Bh is not None else 1) + 8 * n + 8 * n
    d2h = 8 * n

    peak, peak_kind = load_peaks()
    top = max(fam_stats.items(), key=lambda kv: kv[1]["ms"]) if fam_stats else None
    roofline = None
    if top:
        name, st = top
        achieved = st["algorithmic_bytes"] / (st["ms"] * 1e-3) / 1e9 if st["ms"] > 0 else 0.0
        traffic, traffic_note = ncu_traffic(name)
        roofline = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_note,
                    "peak_source": peak_kind,
                    "launches_per_step": st["launches"] / max(1, args.steps),
                    "avg_launch_us": st["ms"] * 1e3 / max(1, st["launches"]),
                    "share_of_step": st["ms"] / max(1e-9, sum(step_ms))}

    line = {
        "metric": METRIC, "value": mean_ms / 1e3, "unit": "s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (config generator, seeded b)",
        "config": config_dict(config, size, n, nnz),
        "result": {"iterations": its, "converged": conv, "levels": levels,
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
        "e2e": {"value": e2e_mean / 1e3, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(round(launches)),
        "roofline": roofline,
        "kernel_families": fam_stats,
        "warmup_family_ms_per_step": {name: round(ms / max(1, args.warmup), 3) for ms, f, name, l, by in fams if l},
        # achieved algorithmic GB/s per family over the warm-up steps (every launch event-timed)
        "family_rooflines": {name: {"ms_per_step": round(ms / max(1, args.warmup), 3),
                                    "achieved_gbs": round(by / (ms * 1e-3) / 1e9, 1),
                                    "frac": round(by / (ms * 1e-3) / 1e9 / peak, 4)}
                             for ms, f, name, l, by in fams if l and by > 0 and ms > 0},
        "clocks": clocks,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            sample, t_cal = cpu_sample("port", config, size, 1, args.cpu_budget / 8, args.max_restarts)
            ts, tv, cits, cconv, clev = oracle_run("port", config, sample, args.max_restarts)
            line["cpu_baseline"] = {"value": scaled_value(ts + tv, config, size, sample), "unit": "s", "cores": 1,
                                    "kind": "port",
                                    "sample": f"config {config} at {sample}^2 ({dofs(config, sample)} DOFs): one "
                                              f"setup+solve of the CPU restatement (oracle/rnamg_port.cpp, single "
                                              f"thread) in {ts + tv:.2f}s, scaled by the DOFs ratio "
                                              f"{dofs(config, size) / dofs(config, sample):.3f}",
                                    "sample_setup_s": ts, "sample_solve_s": tv, "sample_iterations": cits,
                                    "sample_converged": cconv}
        except Exception as e:  # the GPU number stands on its own
            line["cpu_baseline"] = {"value": None, "unit": "s", "cores": 1, "kind": "port", "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
