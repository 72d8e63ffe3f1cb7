"""Throughput of the general-geometry 2D path on a large curved mesh built
here (no reference needed): an n x n box with k_geo = 2 mapping nodes, warped
by a smooth map, wrapped as a reference-like Mesh (faces from the box
connectivity).  Usage: python profiles/general_throughput.py [n] [k]"""
import sys
from types import SimpleNamespace
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.basis import gll_nodes
from paper_1607_01323_b200.general import GeneralSpace2D
from paper_1607_01323_b200.spaces import DgSpace

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
box = M.build_box_mesh(((0, 1), (0, 1)), (n, n))
ref = DgSpace(box, k)
em, sm, ep, sp = ref.interior_faces()
kg = 2
xi = 0.5 * (gll_nodes(kg) + 1.0)
ne = n * n
e = np.arange(ne)
ix, iy = e % n, e // n
X = (ix[None, :, None] + xi[None, None, :]) / n + 0 * xi[:, None, None]
Y = (iy[None, :, None] + xi[:, None, None]) / n + 0 * xi[None, None, :]
s = np.sin(np.pi * X) * np.sin(np.pi * Y)
geom = np.stack([X + 0.05 * s, Y - 0.04 * s])               # (2, mg, ne, mg)
bel, bsl, btag = [], [], []
for side, (sel, slot) in enumerate([(ix == 0, 0), (ix == n - 1, 1), (iy == 0, 2), (iy == n - 1, 3)]):
    bel.append(e[sel]); bsl.append(np.full(sel.sum(), slot)); btag.append(np.full(sel.sum(), side))
mesh = SimpleNamespace(geom_degree=kg, geom_nodes=geom,
                       interior=SimpleNamespace(em=em, sm=sm, ep=ep, sp=sp, flip=np.zeros(em.size, bool)),
                       boundary=SimpleNamespace(elem=np.concatenate(bel), slot=np.concatenate(bsl),
                                                tag=np.concatenate(btag)),
                       tag_names=["xmin", "xmax", "ymin", "ymax"], n_elements=ne)
space = GeneralSpace2D(mesh, k)
bcs = ops.BoundarySpec({"xmin": ops.DirichletBC(None), "xmax": ops.NeumannBC(None, None),
                        "ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(space)
p = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda")
u = torch.rand(2 * space.n_dofs, dtype=torch.float64, device="cuda")


def t(f, reps=20):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for name, f, nd in (("laplace", lambda: ops.apply_pressure_laplace(space, p, bcs), space.n_dofs),
                    ("mass", lambda: ops.mass_apply(space, p), space.n_dofs),
                    ("helmholtz", lambda: ops.apply_viscous_helmholtz(space, u, 10.0, 0.01, bcs), 2 * space.n_dofs),
                    ("convective", lambda: ops.eval_convective_rhs(space, bcs, [u], (1.0,), (0.0,), 0.0), 2 * space.n_dofs)):
    ms = t(f)
    print(f"general 2D {n}x{n} Q{k} {name:11s} {ms:8.3f} ms {nd / ms / 1e6:8.2f} GDoF/s")
cart = ops.BoundarySpec({"xmin": ops.DirichletBC(None), "xmax": ops.NeumannBC(None, None),
                         "ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(ref)
pc = torch.rand(ref.n_dofs, dtype=torch.float64, device="cuda")
ms = t(lambda: ops.apply_pressure_laplace(ref, pc, cart))
print(f"Cartesian 2D {n}x{n} Q{k} laplace     {ms:8.3f} ms {ref.n_dofs / ms / 1e6:8.2f} GDoF/s")
