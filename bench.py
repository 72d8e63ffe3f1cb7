#!/usr/bin/env python
"""Benchmark of the matrix-free DG hot path (BASELINE.json metric).

Headline: SIP Laplace vmult DoF/s (fp64) on BASELINE config 5 -- unit cube,
128^3 Cartesian cells, Q4 (262,144,000 DoFs), walls -- split into x-slabs
across N GPUs (strong scaling, NCCL halo exchange overlapped with interior
cells).  A "step" is one vmult over the whole mesh.  Inputs are larger than
L2 (2.1 GB per vector), so no L2 flush is needed between steps.

Also reported on the same JSON line (rank 0):
  roofline      HBM roofline of the vmult kernel (16 B/DoF algorithmic)
  fp64          fp64 issue-rate view of the same kernel (flop count by design)
  e2e           the same metric through the public API with host buffers
                (pinned H2D of the input + D2H of the result every step)
  cg            BASELINE config 2: Chebyshev(5)-Jacobi PCG to 1e-10 on
                32^3 Q4 (N=1 only)
  cpu_baseline  the numpy oracle (restated reference algorithm) on a
                bounded sample, on this host (N=1, rank 0)
  clocks        SM clocks / throttle reasons sampled (NVML) during the
                timed region

--impl reference: the reference algorithm on the host CPU (numpy port in
oracle/, all host threads), same metric, bounded sample per step.
"""

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6553.3
BYTES_PER_DOF = 16.0          # read src + write dst, fp64
# fp64 instruction count per DoF of laplace_vmult_kernel:
# 7 sweeps x n FMA + face terms; flops = 2 per FMA
FMA_PER_DOF = {n: 7 * n + 18 for n in range(2, 9)}

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake", 0x100: "display_clocks"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cells", type=int, default=128, help="cells per axis (C5: 128)")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--no-cg", action="store_true")
    ap.add_argument("--no-step", action="store_true", help="skip the config-4 time-step timing")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sweep", action="store_true",
                    help="also print the Q2-Q7 degree sweep at 64^3 (extra lines)")
    return ap.parse_args()


class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons in a thread."""

    def __init__(self, index, period=0.02):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        r = [name for bit, name in REASONS.items() if self.reasons & bit]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples), "reasons": r}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


def ncu_summary(k, kernel):
    """Committed ncu --set full summary of the headline vmult kernel at degree
    k (profiles/ncu_laplace.json, written by profiles/r02/ncu_to_summary.py):
    DRAM bytes per launch, fp64 instruction counts per DoF.  Used only if it
    was captured on the kernel this run launches (``kernel`` =
    dg_laplace_kernel_name); otherwise {} -- a stale capture is never reported."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_laplace.json")) as f:
            e = json.load(f).get(f"k{k}", {})
    except Exception:
        return {}
    return e if e.get("kernel") == kernel else {}


def fp64_peak_measured():
    """Measured fp64 DFMA peak (profiles/fp64_peak.cu -> fp64_peak.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            return float(json.load(f)["dfma_tflops"]), "measured DFMA peak (profiles/fp64_peak.json)"
    except Exception:
        return None, None


def oracle_sample(k, cells, threads_all):
    """Reference algorithm (numpy port in oracle/) on a bounded sample:
    cells^3 box, walls, Q_k; returns (DoF/s, dofs, seconds per vmult)."""
    import numpy as np
    from oracle import dg_oracle as O
    m = O.build_box_mesh(((0, 1),) * 3, (cells,) * 3)
    sp = O.DgSpace(m, k)
    b = O.BoundarySpec({t: O.zero_dirichlet(3) for t in m.tag_names}).resolve(sp)
    p = np.random.default_rng(4).uniform(-1, 1, sp.field_shape())
    O.apply_pressure_laplace(sp, p, b)
    return sp, b, p


def run_reference(args, rank, world):
    """--impl reference: the reference's algorithm on the host CPU."""
    if rank != 0:
        return
    import numpy as np
    try:
        import threadpoolctl
        threadpoolctl.threadpool_limits(os.cpu_count())
    except Exception:
        pass
    from oracle import dg_oracle as O
    # bounded sample: the largest box whose K steps fit in ~2.5 minutes
    for cells in ((24, 16, 12, 8) if args.k <= 4 else (16, 12, 8)):
        sp, b, p = oracle_sample(args.k, cells, True)
        t1 = time.perf_counter()
        O.apply_pressure_laplace(sp, p, b)
        if (args.steps + args.warmup) * (time.perf_counter() - t1) <= 150.0:
            break
    for _ in range(args.warmup):
        O.apply_pressure_laplace(sp, p, b)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.apply_pressure_laplace(sp, p, b)
    dt = time.perf_counter() - t0
    val = p.size * args.steps / dt
    cores = len(os.sched_getaffinity(0))
    line = {
        "impl": "reference", "metric": "SIP Laplace vmult DoF/s (fp64)", "value": val,
        "unit": "DoF/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C5-shaped SIP Laplace vmult sample: {cells}^3 cells, Q{args.k}, "
                               f"walls, uniform[-1,1] seed 4 (numpy port of the reference "
                               f"algorithm; the reference package itself is 2D-only)",
                   "cells": cells, "k": args.k},
        "cpu_baseline": {"value": val, "unit": "DoF/s", "cores": cores, "kind": "port",
                         "sample": f"{cells}^3 Q{args.k} vmult x {args.steps}"},
        "e2e": {"value": val, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(k):
    """Oracle port (restated reference algorithm) on the host: 1 BLAS thread
    (the reference tests' setting) and all host threads, ~10 s each."""
    import threadpoolctl
    from oracle import dg_oracle as O
    cells = 24 if k <= 4 else 16
    sp, b, p = oracle_sample(k, cells, False)
    res = {}
    for label, threads in (("one", 1), ("all", len(os.sched_getaffinity(0)))):
        with threadpoolctl.threadpool_limits(threads):
            O.apply_pressure_laplace(sp, p, b)
            reps, t0 = 0, time.perf_counter()
            while time.perf_counter() - t0 < 10.0:
                O.apply_pressure_laplace(sp, p, b)
                reps += 1
            res[label] = (p.size * reps / (time.perf_counter() - t0), threads, reps)
    v1, _, r1 = res["one"]
    va, ca, ra = res["all"]
    return {"value": v1, "unit": "DoF/s", "cores": 1, "kind": "port",
            "sample": f"{cells}^3 cells Q{k} walls vmult x {r1} (numpy port, 1 thread)",
            "all_cores": {"value": va, "unit": "DoF/s", "cores": ca,
                          "sample": f"{cells}^3 cells Q{k} walls vmult x {ra} (numpy port, "
                                    f"{ca} BLAS threads)"}}


def run_c4_step(nsteps=5, mg_precision="fp64"):
    """BASELINE config 4: dual-splitting steps on the 64 x 32 x 32 Q3 channel
    (y graded 1.8, periodic x/z, walls), nu = 1/180, dt = 1e-3, BDF2, V4,
    u0 = (1 - y^2, 0, 0) + 0.1 U(-1,1) (seed 3), history [u0, u0].  The first
    two steps are warm-up (lazy loading of the kernel modules they touch
    first, graph capture of the V-cycle); the median of the rest is
    reported, every step is listed.  mg_precision "fp32": the paper's
    single-precision V-cycle inside the fp64 pressure CG,
    reported beside the fp64 headline, not instead of it."""
    import numpy as np
    import torch
    from paper_1607_01323_b200 import multigrid as MG, operators as ops, stepper as S
    from paper_1607_01323_b200.spaces import DgSpace
    meshes = MG.box_mesh_hierarchy(((0, 2 * np.pi), (-1, 1), (0, np.pi)), (2, 1, 1), 5,
                                   grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
    spaces = [DgSpace(m, 3) for m in meshes]
    spec = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)})
    cfg = S.StepConfig(dt=1e-3, nu=1 / 180, J=2, variant=ops.VariantConfig("V4"),
                       mg_precision=mg_precision)
    vc = S.VelocityCorrection(spaces, spec, cfg)
    x, y, z = spaces[-1].node_coords()
    rng = np.random.default_rng(3)
    u0 = np.stack([1 - y ** 2, 0 * y, 0 * y]) + 0.1 * rng.uniform(-1, 1, (3,) + y.shape)
    u0 = torch.as_tensor(u0.ravel(), device="cuda")
    w0 = ops.compute_vorticity(spaces[-1], u0)
    hu, hp, hw = [u0, u0], [], [w0, w0]
    steps = []
    for n in range(nsteps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = vc.step(hu, hp, hw, n * 1e-3)
        torch.cuda.synchronize()
        steps.append({"ms": 1e3 * (time.perf_counter() - t0), "substep_ms": r.times_ms,
                      "iterations": r.iters})
        hu, hp, hw = [r.u, hu[0]], [r.p] + hp[:1], [r.w, hw[0]]
    return {"config": "C4: 64x32x32 Q3 channel, y graded 1.8, nu 1/180, dt 1e-3, BDF2, V4 "
                      "(zeta* = 1, CFL = 1), MG-PCG pressure, M^-1-PCG projection/viscous",
            "velocity_dofs": 3 * spaces[-1].n_dofs, "ms_per_step_steady": float(
                np.median([s["ms"] for s in steps[2:]])) if nsteps > 2 else steps[-1]["ms"],
            "steps": steps}


def run_degree_sweep(peak_gbs):
    """C5 degree sweep: SIP Laplace vmult at 64^3 cells,
    Q2..Q7, walls as C1; DoF/s and the HBM roofline fraction at 16 B/DoF
    (CUDA events, 20 reps after warm-up; inputs > L2 from Q3 up)."""
    import torch
    from paper_1607_01323_b200 import mesh as M, operators as ops
    from paper_1607_01323_b200.spaces import DgSpace
    out = {}
    mesh = M.build_box_mesh(((0, 1),) * 3, (64, 64, 64))
    for k in range(2, 8):
        space = DgSpace(mesh, k)
        bcs = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()}).resolve(space)
        x = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        f = lambda: ops.apply_pressure_laplace(space, x, bcs)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        dps = space.n_dofs / ms * 1e3
        out[f"Q{k}"] = {"dofs": space.n_dofs, "ms": ms, "dof_per_s": dps,
                        "hbm_frac": dps * 16.0 / (peak_gbs * 1e9)}
        del x, y
    return out


def run_small_configs():
    """BASELINE configs 1 and 3 (latency / fp64-heavy cases, not roofline
    configs): C1 8^3 Q3 walls Laplace vmult with both wall kinds; C3
    convective term 32^3 Q5 periodic [0, 2pi]^3 Taylor-Green + 1e-2 noise
    (seed 2), n_q = 8 (reference rule) and 9 (BASELINE literal)."""
    import numpy as np
    import torch
    from paper_1607_01323_b200 import mesh as M, operators as ops
    from paper_1607_01323_b200.spaces import DgSpace

    def timeit(f, reps=50):
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out = {}
    mesh = M.build_box_mesh(((0, 1),) * 3, (8, 8, 8))
    space = DgSpace(mesh, 3)
    p = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, space.n_dofs), device="cuda")
    for kind, bc in (("dirichlet", ops.DirichletBC(None)), ("neumann", ops.NeumannBC(None, None))):
        bcs = ops.BoundarySpec({t: bc for t in mesh.boundary_tags()}).resolve(space)
        ms = timeit(lambda: ops.apply_pressure_laplace(space, p, bcs))
        out[f"C1_{kind}_walls"] = {"dofs": space.n_dofs, "ms": ms, "dof_per_s": space.n_dofs / ms * 1e3}
    mesh = M.build_box_mesh(((0, 2 * np.pi),) * 3, (32, 32, 32), periodic=(True, True, True))
    for nq in (8, 9):
        space = DgSpace(mesh, 5, n_q_over=nq)
        x, y, z = space.node_coords()
        rng = np.random.default_rng(2)
        u = np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z), 0 * z])
        u = u + 1e-2 * rng.uniform(-1, 1, u.shape)
        ud = torch.as_tensor(u.ravel(), device="cuda")
        bcs = ops.BoundarySpec({}).resolve(space)
        ms = timeit(lambda: ops.eval_convective_rhs(space, bcs, [ud], (1.0,), (0.0,), 0.0), 10)
        out[f"C3_convective_nq{nq}"] = {"velocity_dofs": 3 * space.n_dofs, "ms": ms,
                                       "dof_per_s": 3 * space.n_dofs / ms * 1e3,
                                       "bytes_per_dof": 16.0}
    return out


def run_slab_emulation(n, k, t1_ms, cg1_ms=None):
    """Per-rank compute of the C5 x-slab vmult at P = 2, 4, 8 on ONE GPU: an
    interior slab of the 128^3 mesh with its ghost face traces in device
    buffers (what the NCCL exchange delivers), timed as the production
    split vmult -- whole slab on zero ghost traces (the part that overlaps
    the exchange) + the ghost-trace lifts.  Communication is not included
    (payload and the NVLink time it needs at 900 GB/s are reported beside);
    the compute-only efficiency is T1 / (P T_P)."""
    import ctypes
    import torch
    from paper_1607_01323_b200 import mesh as M, _lib
    from paper_1607_01323_b200.parallel import SlabPartition
    from paper_1607_01323_b200.spaces import DeviceContext
    from paper_1607_01323_b200.operators import ctypes_ptr
    P = lambda t: ctypes_ptr(t.data_ptr())
    out = {}
    mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n))
    kinds = (_lib.BC_VELOCITY_DIRICHLET,) * 6
    st = ctypes_ptr(torch.cuda.current_stream().cuda_stream)
    for nranks in (2, 4, 8):
        part = SlabPartition(n, nranks, False)
        x0, x1 = part.range(1)
        c = DeviceContext(mesh, k, kinds, 0, (x0, x1))
        cnt = ctypes.c_int64()
        _lib.call("dg_halo_count", c.handle, ctypes.byref(cnt))
        nloc = (x1 - x0) * n * n * (k + 1) ** 3
        src = torch.rand(nloc, dtype=torch.float64, device="cuda")
        dst = torch.empty_like(src)
        rcv = [torch.rand(cnt.value, dtype=torch.float64, device="cuda") for _ in range(2)]
        _lib.call("dg_halo_attach", c.handle, P(rcv[0]), P(rcv[1]))
        ts = []
        for ph in (1, 2):
            f = lambda: _lib.call("dg_laplace_vmult_split", c.handle, P(src), P(dst), 1.0, ph, st)
            f()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(20):
                    f()
                b.record()
                torch.cuda.synchronize()
                best = min(best, a.elapsed_time(b) / 20)
            ts.append(best)
        tp = ts[0] + ts[1]
        halo_bytes = 2 * cnt.value * 8  # both neighbours, one direction
        out[f"P{nranks}"] = {"slab_cells": [x1 - x0, n, n], "whole_slab_ms": ts[0],
                             "ghost_lift_ms": ts[1], "rank_vmult_ms": tp,
                             "compute_efficiency": t1_ms / (nranks * tp),
                             "halo_bytes_per_rank": halo_bytes,
                             "nvlink_ms_at_900GBs": halo_bytes / 2 / 900e9 * 1e3}
        if cg1_ms is not None:
            # the rank's kernels of one SlabPCG Jacobi iteration (projected
            # operator as in cg_iteration_c5): split vmult with its dot shares,
            # x / r / z update with r.z, p update; all-reduces (two of <= 3
            # doubles) and the exchange excluded
            x, r, z, dg = (torch.rand(nloc, dtype=torch.float64, device="cuda") + 0.5
                           for _ in range(4))
            scal = torch.tensor([1.0, 2.0, 0.0, 0.0, 1.0, 0, 0, 0], dtype=torch.float64,
                                device="cuda")
            s3 = torch.zeros(3, dtype=torch.float64, device="cuda")

            def it():
                for ph in (1, 2):
                    _lib.call("dg_laplace_vmult_split_dots", c.handle, P(src), P(dst), 1.0, ph,
                              P(s3), st)
                _lib.call("dg_cg_update", c.handle, P(x), P(r), P(src), P(dst), P(scal), 1, P(dg),
                          P(z), P(s3), st)
                _lib.call("dg_cg_pupdate", c.handle, P(src), P(z), P(scal), st)
                scal[0] = 1.0  # keep beta bounded over the repetitions
            it()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(10):
                    it()
                b.record()
                torch.cuda.synchronize()
                best = min(best, a.elapsed_time(b) / 10)
            out[f"P{nranks}"]["rank_cg_iteration_ms"] = best
            out[f"P{nranks}"]["cg_compute_efficiency"] = cg1_ms / (nranks * best)
            del x, r, z, dg
        del c, src, dst, rcv
    out["note"] = ("one GPU, interior slab, ghost traces from device buffers; communication "
                   "excluded (overlapped with the whole-slab phase in the product)")
    return out


def run_cg(dist_on):
    """BASELINE config 2: 32^3, Q4, periodic x,z, walls y, pure Neumann,
    rhs = zero_mean_project_dual(M (sin 2pi x cos pi y sin 2pi z + 1e-3 N(0,1),
    seed 1)), Chebyshev(5, 20) over Jacobi, rel_tol 1e-10."""
    import numpy as np
    import torch
    from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol
    from paper_1607_01323_b200.spaces import DgSpace
    mesh = M.build_box_mesh(((0, 1),) * 3, (32, 32, 32), periodic=(True, False, True))
    space = DgSpace(mesh, 4)
    bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None),
                            "ymax": ops.DirichletBC(None)}).resolve(space)
    xn = space.node_coords()
    f = np.sin(2 * np.pi * xn[0]) * np.cos(np.pi * xn[1]) * np.sin(2 * np.pi * xn[2])
    f = f + 1e-3 * np.random.default_rng(1).standard_normal(f.shape)
    b = sol.zero_mean_project_dual(space, ops.mass_apply(space, torch.as_tensor(
        f.ravel(), device="cuda")))
    diag = ops.laplace_diagonal(space, bcs)
    lmax = sol.lanczos_lambda_max(space, bcs, diag, project=True)
    cfg = sol.ChebyshevConfig(5, 20.0, lmax)
    sol.laplace_pcg(space, bcs, b, project_dual=True, cheb=cfg, diag=diag, rel_tol=1e-10,
                    max_iter=5)  # warm-up
    dt = 1e30
    for _ in range(2):  # whole solves, wall clock; the faster of two (one-time set-up in the first)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, st = sol.laplace_pcg(space, bcs, b, project_dual=True, cheb=cfg, diag=diag,
                                rel_tol=1e-10, max_iter=5000)
        torch.cuda.synchronize()
        dt = min(dt, time.perf_counter() - t0)
    out = {"config": "C2: 32^3 Q4 periodic x,z / walls y, Chebyshev(5,20)-Jacobi PCG, rel_tol 1e-10",
           "dofs": space.n_dofs, "iterations": st.iterations, "converged": st.converged,
           "solve_ms": 1e3 * dt, "ms_per_iteration": 1e3 * dt / max(st.iterations, 1),
           "dof_per_s_per_iteration": space.n_dofs * st.iterations / dt,
           "lambda_max": lmax}
    # the reference's actual Poisson preconditioner: geometric multigrid
    # V-cycle (multigrid.py), levels 4^3 .. 32^3, same right-hand side
    from paper_1607_01323_b200 import multigrid as MG
    meshes = MG.box_mesh_hierarchy(((0, 1),) * 3, (4, 4, 4), 3, periodic=(True, False, True))
    spaces = [DgSpace(m, 4) for m in meshes]
    spec = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)})
    mg = MG.MultigridHierarchy(spaces, spec, project=sol.zero_mean_project)
    bb = b.reshape(-1)
    MG.laplace_pcg_mg(mg, bb, project_dual=True, rel_tol=1e-10, max_iter=3)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    xm, stm = MG.laplace_pcg_mg(mg, bb, project_dual=True, rel_tol=1e-10, max_iter=200)
    torch.cuda.synchronize()
    dtm = time.perf_counter() - t0
    out["multigrid"] = {"levels": mg.n_levels, "coarse_iters": mg.levels[0].coarse_iters,
                        "iterations": stm.iterations, "converged": stm.converged,
                        "solve_ms": 1e3 * dtm,
                        "rel_diff_vs_chebyshev": float((xm.reshape(-1) - x.reshape(-1)).norm()
                                                       / x.reshape(-1).norm())}
    # the paper's single-precision V-cycle inside the fp64 CG
    mg32 = MG.MultigridHierarchy(spaces, spec, project=sol.zero_mean_project, precision="fp32")
    MG.laplace_pcg_mg(mg32, bb, project_dual=True, rel_tol=1e-10, max_iter=3)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x32, st32 = MG.laplace_pcg_mg(mg32, bb, project_dual=True, rel_tol=1e-10, max_iter=200)
    torch.cuda.synchronize()
    dt32 = time.perf_counter() - t0
    out["multigrid_fp32"] = {"iterations": st32.iterations, "converged": st32.converged,
                             "solve_ms": 1e3 * dt32,
                             "rel_diff_vs_fp64_mg": float((x32 - xm.reshape(-1)).norm()
                                                          / xm.reshape(-1).norm())}
    return out


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import numpy as np
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1607_01323_b200 import mesh as M, _lib
    from paper_1607_01323_b200.parallel import SlabLaplace

    n, k = args.cells, args.k
    mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n))
    kinds = (_lib.BC_VELOCITY_DIRICHLET,) * 6
    op = SlabLaplace(mesh, k, kinds, rank, world)
    nd = op.n_dofs
    total = mesh.n_elements * (k + 1) ** 3
    g = torch.Generator(device="cuda").manual_seed(4 + rank)
    src = torch.rand(nd, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    dst = torch.empty_like(src)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        op.vmult(src, dst)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            op.vmult(src, dst)
        e1.record()
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    ms_step = ms / args.steps
    value = total / (ms_step * 1e-3)

    # end to end through the public API: pinned host in -> device -> host out
    e2e = None
    if not args.no_e2e and world == 1:
        # the public call with host buffers: ops.apply_pressure_laplace on a
        # pinned CPU tensor (dg_laplace_vmult_host: chunked H2D / vmult / D2H
        # overlapped on three streams)
        from paper_1607_01323_b200 import operators as ops
        from paper_1607_01323_b200.spaces import DgSpace
        space = DgSpace(mesh, k)
        bcs = ops.BoundarySpec({t: ops.DirichletBC(None)
                                for t in mesh.boundary_tags()}).resolve(space)
        K2 = max(3, min(args.steps, 10))
        h_in = torch.empty(nd, dtype=torch.float64, pin_memory=True)
        h_in.copy_(src.cpu())
        for _ in range(2):
            h_out = ops.apply_pressure_laplace(space, h_in, bcs)
        same = bool(torch.equal(h_out, dst.cpu()))  # dst = the device path's result
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(K2):
            h_out = ops.apply_pressure_laplace(space, h_in, bcs)
        f1.record()
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1)
        e2e = {"value": total / (ems / K2 * 1e-3), "unit": "DoF/s",
               "h2d_bytes_per_step": 8 * total, "d2h_bytes_per_step": 8 * total,
               "ms_per_step": ems / K2, "steps": K2,
               "api": "operators.apply_pressure_laplace(space, pinned CPU tensor, bcs)",
               "bitwise_equal_to_device_path": same}
    elif not args.no_e2e:
        K2 = max(3, min(args.steps, 10))
        h_in = torch.empty(nd, dtype=torch.float64, pin_memory=True)
        h_in.copy_(src.cpu())
        h_out = torch.empty(nd, dtype=torch.float64, pin_memory=True)
        d_in = torch.empty_like(src)
        for _ in range(2):
            d_in.copy_(h_in, non_blocking=True)
            op.vmult(d_in, dst)
            h_out.copy_(dst, non_blocking=True)
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(K2):
            d_in.copy_(h_in, non_blocking=True)
            op.vmult(d_in, dst)
            h_out.copy_(dst, non_blocking=True)
        f1.record()
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        e2e = {"value": total / (ems / K2 * 1e-3), "unit": "DoF/s",
               "h2d_bytes_per_step": 8 * total, "d2h_bytes_per_step": 8 * total,
               "ms_per_step": ems / K2, "steps": K2}

    # C5 CG iteration on every rank count: parallel.SlabPCG
    # (the reference pcg with point-Jacobi preconditioning, pure-Neumann
    # projected operator as the walls make it): slab vmult with overlapped
    # halo exchange, dg_cg_dots, NCCL all-reduce, fused x/r/z update with r.z,
    # NCCL all-reduce, host stop test, p update -- fixed iteration count
    cgi = None
    if not args.no_cg:
        from paper_1607_01323_b200.parallel import SlabPCG
        solver = SlabPCG(op, op.diagonal(), cheb=None, project_dual=True)
        solver.start(src, rel_tol=0.0)
        for _ in range(3):
            solver.step()
        torch.cuda.synchronize()
        barrier()
        KC = 20
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(KC):
            solver.step()
        c1.record()
        torch.cuda.synchronize()
        cms = c0.elapsed_time(c1)
        if world > 1:
            t = torch.tensor([cms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            cms = t.item()
        cgi = {"config": f"C5: {n}^3 Q{k} walls, Jacobi-PCG iteration (parallel.SlabPCG): x-slab "
                         f"vmult with p.Lp / sum(Lp) / p.w formed in its epilogue "
                         f"(dg_laplace_vmult_dots / _split_dots), overlapped face-trace halo "
                         f"exchange + 2 NCCL all-reduces + fused vector kernels + host stop "
                         f"test, {world} GPU(s)",
               "iterations": KC, "ms_per_iteration": cms / KC,
               "dof_per_s_per_iteration": total / (cms / KC * 1e-3),
               "bytes_per_dof_algorithmic": 96,
               "hbm_frac_of_96B_per_dof": total * 96 / (cms / KC * 1e-3) / 1e9 / hbm_peak()[0],
               "vmult_share": ms_step / (cms / KC)}
        del solver

    cg = None
    if rank == 0 and world == 1 and not args.no_cg:
        cg = run_cg(False)
    step = None
    if rank == 0 and world == 1 and not args.no_step:
        step = run_c4_step()
        s32 = run_c4_step(4, "fp32")
        step["mg_fp32"] = {"ms_per_step_steady": s32["ms_per_step_steady"],
                           "iterations": [x["iterations"] for x in s32["steps"]],
                           "note": "the paper's single-precision V-cycle in the fp64 CG"}
    small = dsweep = None
    if rank == 0 and world == 1 and not args.no_step:
        small = run_small_configs()
        dsweep = run_degree_sweep(hbm_peak()[0])
    slab_emu = None
    if rank == 0 and world == 1 and not args.no_step:
        try:
            slab_emu = run_slab_emulation(n, k, ms_step, cgi["ms_per_iteration"] if cgi else None)
        except Exception as exc:  # reported, never fatal for the headline line
            slab_emu = {"error": repr(exc)[:200]}
    sweep = []
    if rank == 0 and world == 1 and args.sweep:
        sweep = run_sweep()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(k)

    if rank == 0:
        import ctypes
        peak, peak_kind = hbm_peak()
        per_rank_dofs = nd
        achieved = per_rank_dofs * BYTES_PER_DOF / (ms_step * 1e-3) / 1e9
        clocks = clk.summary()
        kbuf = ctypes.create_string_buffer(128)
        _lib.call("dg_laplace_kernel_name", op.ctx.handle, kbuf, 128)
        kernel = kbuf.value.decode()
        prof = ncu_summary(k, kernel)
        fma = FMA_PER_DOF.get(k + 1)
        flop = prof.get("flop_per_dof") or (2 * fma if fma else None)
        sm_mhz = clocks["sm_mhz"] or 1965.0
        fp64_peak, fp64_kind = fp64_peak_measured()
        if fp64_peak is None:
            fp64_peak = 148 * 64 * 2 * sm_mhz * 1e6 / 1e12
            fp64_kind = "nominal 64 DFMA/clk/SM x 148 SMs x median SM clock"
        fp64_ach = per_rank_dofs * flop / (ms_step * 1e-3) / 1e12 if flop else None
        line = {
            "metric": "SIP Laplace vmult DoF/s (fp64)",
            "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: uniform[-1,1] input vector (torch generator seed 4+rank)",
            "config": {"workload": f"C5: SIP Laplace vmult, unit cube {n}^3 Cartesian cells, "
                                   f"Q{k} DG (GLL nodes, {k + 1} Gauss points), velocity-Dirichlet "
                                   f"walls, x-slabs over {world} GPU(s)",
                       "cells": n, "k": k, "dofs": total, "parallelism": f"x-slabs{world}",
                       "l2": "inputs (8 B/DoF x dofs) larger than L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": (prof.get("dram_bytes_per_launch") / world
                                     if prof and n == 128 and world == 1 else None),
                         "traffic_source": (prof.get("source") if prof else
                                            "no ncu capture of this kernel committed"),
                         "peak_kind": peak_kind,
                         "algorithmic_bytes_per_dof": BYTES_PER_DOF,
                         "kernel": kernel},
            "fp64": {"flop_per_dof": flop,
                     "fp64_inst_per_dof": prof.get("fp64_inst_per_dof"),
                     "flop_source": ("ncu sass dfma/dadd/dmul counts of this kernel "
                                     "(profiles/ncu_laplace.json)"
                                     if prof.get("flop_per_dof") else "model 2 x (7n + 18)"),
                     "achieved_tflops": fp64_ach,
                     "peak_tflops": fp64_peak,
                     "frac": (fp64_ach / fp64_peak) if flop else None,
                     "peak_kind": fp64_kind},
            "gpu_launches": args.steps * (1 if world == 1 else 2),
            "clocks": clocks,
        }
        if e2e:
            line["e2e"] = e2e
        if cgi:
            line["cg_iteration_c5"] = cgi
        if cg:
            line["cg"] = cg
        if step:
            line["c4_step"] = step
        if small:
            line["configs"] = small
        if dsweep:
            line["degree_sweep_64cubed"] = dsweep
        if slab_emu:
            line["slab_emulation_1gpu"] = slab_emu
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
        for s in sweep:
            print(json.dumps(s), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sweep():
    """Degree sweep Q2-Q7 at 64^3 cells on one GPU (config 5 second part)."""
    import torch
    from paper_1607_01323_b200 import mesh as M, _lib
    from paper_1607_01323_b200.parallel import SlabLaplace
    out = []
    mesh = M.build_box_mesh(((0, 1),) * 3, (64, 64, 64))
    peak, _ = hbm_peak()
    for k in range(2, 8):
        op = SlabLaplace(mesh, k, (_lib.BC_VELOCITY_DIRICHLET,) * 6, 0, 1)
        src = torch.rand(op.n_dofs, dtype=torch.float64, device="cuda")
        dst = torch.empty_like(src)
        for _ in range(5):
            op.vmult(src, dst)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        e0.record()
        for _ in range(reps):
            op.vmult(src, dst)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        dofs = op.n_dofs
        out.append({"sweep": "laplace_vmult_64cubed", "k": k, "dofs": dofs, "ms": ms,
                    "dof_per_s": dofs / (ms * 1e-3),
                    "hbm_frac": dofs * BYTES_PER_DOF / (ms * 1e-3) / 1e9 / peak})
        del op, src, dst
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
