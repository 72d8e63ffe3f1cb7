"""Diagnostic: fused vs oracle iteration counts of the stepper test cases
(tests/test_gpu_stepper.py setups), with the final residual / tolerance."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from tests.test_gpu_stepper import CASES, setups, initial, dev, host, force
from paper_1607_01323_b200 import stepper as S, operators as ops
from oracle import dg_oracle as O, stepper as OS

for name in CASES:
    for fused in (False, True):
        osp, ospec, gsp, gspec = setups(name)
        bf = force if name == "outflow" else None
        ocfg = OS.StepConfig(dt=1e-3, nu=1 / 180, variant=OS.Variant("V4"), body_force=bf)
        gcfg = S.StepConfig(dt=1e-3, nu=1 / 180, variant=ops.VariantConfig("V4"), body_force=bf)
        ovc = OS.VelocityCorrection(osp, ospec, ocfg, seed_draw=lambda rng, sp: rng.standard_normal(sp.field_shape()))
        gvc = S.VelocityCorrection(gsp, gspec, gcfg, fused=fused)
        u0 = initial(osp[-1])
        ow = O.compute_vorticity(osp[-1], u0)
        ou, op_, ow_h = [u0, u0], [], [ow, ow]
        gu, gp_, gw_h = [dev(u0), dev(u0)], [], [dev(ow), dev(ow)]
        for n in range(2):
            t = n * 1e-3
            ro = ovc.step(ou, op_, ow_h, t)
            rg = gvc.step(gu, gp_, gw_h, t)
            rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
            print(name, "fused" if fused else "plain", n, "oracle", ro.iters, "gpu", rg.iters,
                  "p %.1e u %.1e" % (rel(host(rg.p), ro.p.ravel()), rel(host(rg.u), ro.u.ravel())), flush=True)
            ou, op_, ow_h = [ro.u, ou[0]], [ro.p] + op_[:1], [ro.w, ow_h[0]]
            gu, gp_, gw_h = [rg.u, gu[0]], [rg.p] + gp_[:1], [rg.w, gw_h[0]]
