"""Dual-splitting (velocity-correction) time step on the GPU.

The reference specifies this step (SPEC.md "splitting_scheme"; PAPER.md
Eqs. 37-40, Section 5.1) but ships no code for it; every operator, right-hand
side and solver it is made of is a pinned row of this package:

  (a) convective step   gamma0 u^ = sum alpha_i u^{n-i} + dt M^-1 conv     (Eq. 37)
  (b) pressure Poisson  L p = a(q, u^) + Neumann data + Dirichlet data     (Eq. 38)
      zero-mean projection without outflow, multigrid-preconditioned CG
  (c) projection        (M + tau_D D + tau_C C) u^^ = M u^ + b(v, p)       (Eq. 39)
      element-local CG (V3x) or global CG (V4), inverse-mass preconditioned
  (d) viscous step      (gamma0/dt M - F^nu) u = gamma0/dt M u^^ + bc      (Eq. 40)
      inverse-mass preconditioned CG

Solver initial guesses are order-J extrapolations (Section 5.1).
Vectors are device tensors (element-major); per-substep fields and solver
iteration counts are returned for parity checks and timing.  V2 (HONS,
PAPER.md Eqs. 26-28): (a) yields u^_dt = M^-1 conv, (b) takes the divergence
of u^_dt alone (no 1/dt divergence of the BDF history), and u^ = dt/gamma0
u^_dt + sum alpha_i/gamma0 u^{n-i} is reconstructed before (c).
"""

import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional

from . import operators as ops
from . import solvers as sol
from . import multigrid as MG
from .spaces import _torch

VARIANTS = ("VHW", "V1", "V2", "V3a", "V3b", "V3c", "V4")


def bdf_ex_constants(J):
    """BDF-J / EX-J constants gamma0, alpha_i, beta_i (SPEC.md
    splitting_scheme: bdf_ex_constants)."""
    if J == 1:
        return 1.0, (1.0,), (1.0,)
    if J == 2:
        return 1.5, (2.0, -0.5), (2.0, -1.0)
    if J == 3:
        return 11.0 / 6.0, (3.0, -1.5, 1.0 / 3.0), (3.0, -3.0, 1.0)
    raise ValueError(f"unsupported BDF order J={J}")


@dataclass
class StepConfig:
    dt: float
    nu: float
    J: int = 2
    variant: ops.VariantConfig = field(default_factory=ops.VariantConfig)
    cfl: float = 1.0
    rel_tol_p: float = 1e-8
    rel_tol_v: float = 1e-8
    rel_tol_proj: float = 1e-12
    max_iter: int = 1000
    body_force: Optional[Callable] = None
    mg_precision: str = "fp64"   # "fp32": the paper's single-precision V-cycle


@dataclass
class StepResult:
    u: object
    p: object
    w: object
    uhat: object
    uhh: object
    iters: dict
    times_ms: dict


class VelocityCorrection:
    """One dual-splitting step per call on the finest of ``mg_spaces``
    (nested boxes for the Poisson multigrid).  ``fused`` selects the device
    MG-PCG for the pressure (dg_laplace_pcg_mg, solving for the correction to
    the extrapolated guess) instead of the generic callable PCG."""

    def __init__(self, mg_spaces, bc_spec, cfg: StepConfig, fused: bool = True):
        if cfg.variant.variant not in VARIANTS:
            raise ValueError(f"unsupported variant {cfg.variant.variant!r}")
        self.space = mg_spaces[-1]
        self.cfg, self.fused = cfg, fused
        self.bcs = bc_spec.resolve(self.space)
        self.outflow = self.bcs.has_outflow
        self.tau_scale = (cfg.variant.dt_ref / cfg.dt) if cfg.variant.variant == "V1" else 1.0
        self.g0, self.alpha, self.beta = bdf_ex_constants(cfg.J)
        proj = None if self.outflow else sol.zero_mean_project
        self.mg = MG.MultigridHierarchy(mg_spaces, bc_spec, tau_scale=self.tau_scale, project=proj,
                                        precision=cfg.mg_precision)

    def _pressure(self, rhs, p0):
        cfg, sp, bcs = self.cfg, self.space, self.bcs
        L = lambda p: ops.apply_pressure_laplace(sp, p, bcs, self.tau_scale)
        if self.fused:
            b = rhs if p0 is None else rhs - (L(p0) if self.outflow
                                              else sol.zero_mean_project_dual(sp, L(p0)))
            dp, st = MG.laplace_pcg_mg(self.mg, b, project_dual=not self.outflow,
                                       rel_tol=cfg.rel_tol_p, max_iter=cfg.max_iter)
            return (dp if p0 is None else p0 + dp), st
        op = L if self.outflow else (lambda p: sol.zero_mean_project_dual(sp, L(p)))
        return sol.pcg(op, self.mg.vcycle, rhs, x0=p0, rel_tol=cfg.rel_tol_p,
                       max_iter=cfg.max_iter)

    def step(self, hist_u: List, hist_p: List, hist_w: List, t_n: float) -> StepResult:
        torch = _torch()
        cfg, sp, bcs = self.cfg, self.space, self.bcs
        J, dt, nu, g0 = cfg.J, cfg.dt, cfg.nu, self.g0
        al, be = self.alpha, self.beta
        t_np1 = t_n + dt
        times = [t_n - i * dt for i in range(J)]
        it, tm = {}, {}
        clock = time.perf_counter

        def mark(name, t0):
            torch.cuda.synchronize()
            tm[name] = 1e3 * (clock() - t0)
            return clock()

        t0 = clock()
        # (a) convective step
        conv = ops.eval_convective_rhs(sp, bcs, hist_u[:J], be, times, t_np1, cfg.body_force)
        v2 = cfg.variant.variant == "V2"
        if v2:
            udt = ops.inverse_mass_apply(sp, conv)
            uhat = (dt / g0) * udt + sum((al[i] / g0) * hist_u[i] for i in range(J))
        else:
            uhat = sum(al[i] * hist_u[i] for i in range(J)) + dt * ops.inverse_mass_apply(sp, conv)
            uhat = uhat / g0
        t0 = mark("convective", t0)
        # (b) pressure Poisson
        if v2:
            rhs = ops.eval_divergence_rhs(sp, udt, bcs, 1.0, cfg.variant.a_form)
        else:
            rhs = ops.eval_divergence_rhs(sp, uhat, bcs, g0 / dt, cfg.variant.a_form)
        if bcs.dirichlet:
            rhs = rhs + ops.eval_pressure_neumann_rhs(sp, bcs, hist_u[:J], hist_w[:J], be, nu,
                                                      t_np1, cfg.body_force)
        if bcs.neumann:
            rhs = rhs + ops.gp_dirichlet_rhs(sp, bcs, t_np1, self.tau_scale, like="device").view(
                rhs.shape)
        if not self.outflow:
            rhs = sol.zero_mean_project_dual(sp, rhs)
        if hist_p and len(hist_p) >= J:
            p0 = sum(be[i] * hist_p[i] for i in range(J))
        else:
            p0 = hist_p[0] if hist_p else None
        p, st = self._pressure(rhs, p0)
        it["pressure"] = st.iterations
        t0 = mark("pressure", t0)
        # (c) projection
        rhs = ops.mass_apply(sp, uhat) + ops.eval_pressure_gradient_rhs(sp, p, bcs, dt / g0,
                                                                        cfg.variant.b_form)
        if not cfg.variant.uses_divdiv:
            uhh = ops.inverse_mass_apply(sp, rhs)
            it["projection"] = 0
        else:
            tau_d, tau_c = ops.compute_penalty_parameters(sp, hist_u[0], dt, cfg.cfl, cfg.variant)
            if cfg.variant.local_projection:
                uhh, its, _ = sol.projection_element_pcg(sp, rhs, tau_d, rel_tol=cfg.rel_tol_proj)
                it["projection"] = int(its.max())
            else:
                if self.fused and sp.dim == 3:
                    uhh, st = sol.projection_pcg(sp, rhs, tau_d, tau_c, x0=uhat,
                                                 rel_tol=cfg.rel_tol_proj, max_iter=cfg.max_iter)
                else:
                    uhh, st = sol.pcg(lambda w: ops.apply_projection_operator(sp, w, tau_d, tau_c),
                                      lambda r: ops.inverse_mass_apply(sp, r), rhs, x0=uhat,
                                      rel_tol=cfg.rel_tol_proj, max_iter=cfg.max_iter)
                it["projection"] = st.iterations
        t0 = mark("projection", t0)
        # (d) viscous step
        rhs = (g0 / dt) * ops.mass_apply(sp, uhh)
        if bcs.dirichlet or bcs.neumann:
            rhs = rhs + ops.viscous_rhs_bc(sp, bcs, t_np1, nu, like="device").view(rhs.shape)
        u0 = sum(be[i] * hist_u[i] for i in range(J))
        if self.fused and sp.dim == 3:
            u, st = sol.helmholtz_pcg(sp, bcs, rhs, g0 / dt, nu, x0=u0, rel_tol=cfg.rel_tol_v,
                                      max_iter=cfg.max_iter)
        else:
            u, st = sol.pcg(lambda v: ops.apply_viscous_helmholtz(sp, v, g0 / dt, nu, bcs),
                            lambda r: ops.inverse_mass_apply(sp, r), rhs, x0=u0,
                            rel_tol=cfg.rel_tol_v, max_iter=cfg.max_iter)
        it["viscous"] = st.iterations
        w = ops.compute_vorticity(sp, u)
        mark("viscous", t0)
        return StepResult(u, p, w, uhat, uhh, it, tm)
