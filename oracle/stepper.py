"""Dual-splitting (velocity-correction) time step -- TEST INFRASTRUCTURE.

CPU restatement of the time step the reference specifies but does not ship
(SPEC.md "splitting_scheme", Eqs. 37-40 / Section 5.1): (a) explicit
convective step with the inverse mass, (b) pressure Poisson solve with the
variant's divergence form, consistent Neumann data, pressure-Dirichlet data,
zero-mean projection without outflow, multigrid-preconditioned CG, (c)
projection with the variant's pressure-gradient form and div-div / jump
penalties (element-local CG for V3x, global CG for V4), (d) viscous
Helmholtz solve with inverse-mass preconditioning; solver initial guesses
are order-J extrapolations (Section 5.1).  Built only from the
oracle's operators and solvers (oracle/dg_oracle.py, oracle/multigrid.py),
so each substep's parity with the device step reduces to the already
pinned operators.  V2 (the HONS path, Eqs. 26-28 / SPEC.md
advance_step): the convective step yields u^_dt = M^-1 conv, the Poisson
right-hand side is the divergence of u^_dt alone (the 1/dt divergence of the
BDF history is dropped), and u^ = dt/gamma0 u^_dt + sum alpha_i/gamma0 u^{n-i}
is reconstructed for the projection.
"""

from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import dg_oracle as O
from . import multigrid as OMG


def bdf_ex_constants(J):
    """BDF-J / EX-J constants (SPEC.md splitting_scheme: bdf_ex_constants)."""
    if J == 1:
        return 1.0, (1.0,), (1.0,)
    if J == 2:
        return 1.5, (2.0, -0.5), (2.0, -1.0)
    if J == 3:
        return 11.0 / 6.0, (3.0, -1.5, 1.0 / 3.0), (3.0, -3.0, 1.0)
    raise ValueError(f"unsupported BDF order J={J}")


VARIANTS = ("VHW", "V1", "V2", "V3a", "V3b", "V3c", "V4")


@dataclass
class Variant:
    """operators.py:29-75."""
    variant: str = "V3c"
    zeta_d_star: float = 1.0
    zeta_c_star: float = 1.0
    dt_ref: Optional[float] = None

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unsupported variant {self.variant!r}")

    uses_divdiv = property(lambda s: s.variant in ("V3a", "V3b", "V3c", "V4"))
    uses_jump = property(lambda s: s.variant == "V4")
    a_form = property(lambda s: "weak" if s.variant in ("V3b", "V3c") else "standard")
    b_form = property(lambda s: "weak" if s.variant == "V3c" else "standard")


@dataclass
class StepConfig:
    dt: float
    nu: float
    J: int = 2
    variant: Variant = field(default_factory=Variant)
    cfl: float = 1.0
    rel_tol_p: float = 1e-8
    rel_tol_v: float = 1e-8
    rel_tol_proj: float = 1e-12
    max_iter: int = 1000
    body_force: Optional[Callable] = None


@dataclass
class StepResult:
    u: np.ndarray
    p: np.ndarray
    w: np.ndarray
    uhat: np.ndarray
    uhh: np.ndarray
    iters: dict


class VelocityCorrection:
    def __init__(self, mg_spaces, bc_spec, cfg: StepConfig, seed_draw=None):
        self.space = mg_spaces[-1]
        self.cfg = cfg
        self.bcs = bc_spec.resolve(self.space)
        self.outflow = len(self.bcs.neumann) > 0
        self.tau_scale = (cfg.variant.dt_ref / cfg.dt) if cfg.variant.variant == "V1" else 1.0
        self.g0, self.alpha, self.beta = bdf_ex_constants(cfg.J)
        proj = None if self.outflow else O.zero_mean_project
        self.mg = OMG.MultigridHierarchy(mg_spaces, bc_spec, tau_scale=self.tau_scale,
                                         project=proj, seed_draw=seed_draw)

    def step(self, hist_u: List[np.ndarray], hist_p: List[np.ndarray], hist_w: List[np.ndarray],
             t_n: float) -> StepResult:
        cfg, sp, bcs, dim = self.cfg, self.space, self.bcs, self.space.dim
        J, dt, nu, g0 = cfg.J, cfg.dt, cfg.nu, self.g0
        al, be = self.alpha, self.beta
        t_np1 = t_n + dt
        times = [t_n - i * dt for i in range(J)]
        it = {}
        # (a) convective step (Eq. 37)
        conv = O.eval_convective_rhs(sp, bcs, hist_u[:J], be, times, t_np1, cfg.body_force)
        if cfg.variant.variant == "V2":
            # HONS (Eqs. 26-28): u^_dt (Eq. 26), Poisson rhs -div u^_dt (Eq. 27),
            # u^ reconstructed from u^_dt and the BDF history (Eq. 28)
            udt = O.inverse_mass_apply(sp, conv)
            uhat = (dt / g0) * udt + sum((al[i] / g0) * hist_u[i] for i in range(J))
            rhs = O.eval_divergence_rhs(sp, udt, bcs, 1.0, cfg.variant.a_form)
        else:
            uhat = sum(al[i] * hist_u[i] for i in range(J)) + dt * O.inverse_mass_apply(sp, conv)
            uhat = uhat / g0
            # (b) pressure Poisson (Eq. 38)
            rhs = O.eval_divergence_rhs(sp, uhat, bcs, g0 / dt, cfg.variant.a_form)
        rhs = rhs + O.eval_pressure_neumann_rhs(sp, bcs, hist_u[:J], hist_w[:J], be, nu, t_np1,
                                                cfg.body_force)
        rhs = rhs + O.gp_dirichlet_rhs(sp, bcs, t_np1, self.tau_scale)
        L = lambda p: O.apply_pressure_laplace(sp, p, bcs, self.tau_scale)
        if not self.outflow:
            rhs = O.zero_mean_project_dual(sp, rhs)
            op = lambda p: O.zero_mean_project_dual(sp, L(p))
        else:
            op = L
        if hist_p and len(hist_p) >= J:
            p0 = sum(be[i] * hist_p[i] for i in range(J))
        else:
            p0 = hist_p[0] if hist_p else None
        p, st = O.pcg(op, self.mg.vcycle, rhs, x0=p0, rel_tol=cfg.rel_tol_p, max_iter=cfg.max_iter)
        it["pressure"] = st.iterations
        # (c) projection (Eq. 39)
        rhs = O.mass_apply(sp, uhat) + O.eval_pressure_gradient_rhs(sp, p, bcs, dt / g0,
                                                                    cfg.variant.b_form)
        tau_d = tau_c = None
        if cfg.variant.uses_divdiv:
            tau_d, tau_c = O.compute_penalty_parameters(
                sp, hist_u[0], dt, cfg.cfl, cfg.variant.zeta_d_star, cfg.variant.zeta_c_star,
                True, cfg.variant.uses_jump)
        if not cfg.variant.uses_divdiv:
            uhh = O.inverse_mass_apply(sp, rhs)
            it["projection"] = 0
        elif not cfg.variant.uses_jump:
            uhh, its, _ = O.element_local_pcg(
                lambda w: O.apply_projection_operator(sp, w, tau_d, None),
                lambda r: O.inverse_mass_apply(sp, r), rhs, rel_tol=cfg.rel_tol_proj)
            it["projection"] = int(its.max())
        else:
            uhh, st = O.pcg(lambda w: O.apply_projection_operator(sp, w, tau_d, tau_c),
                            lambda r: O.inverse_mass_apply(sp, r), rhs, x0=uhat,
                            rel_tol=cfg.rel_tol_proj, max_iter=cfg.max_iter)
            it["projection"] = st.iterations
        # (d) viscous step (Eq. 40)
        rhs = (g0 / dt) * O.mass_apply(sp, uhh) + O.viscous_rhs_bc(sp, bcs, t_np1, nu)
        u0 = sum(be[i] * hist_u[i] for i in range(J))
        u, st = O.pcg(lambda v: O.apply_viscous_helmholtz(sp, v, g0 / dt, nu, bcs),
                      lambda r: O.inverse_mass_apply(sp, r), rhs, x0=u0, rel_tol=cfg.rel_tol_v,
                      max_iter=cfg.max_iter)
        it["viscous"] = st.iterations
        w = O.compute_vorticity(sp, u)
        return StepResult(u, p, w, uhat, uhh, it)
