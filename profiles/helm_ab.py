import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace
mesh = M.build_box_mesh(((0, 2*np.pi), (-1, 1), (0, np.pi)), (64, 32, 32), grading=(0, 1.8, 0), periodic=(True, False, True))
space = DgSpace(mesh, 3)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(space)
u = torch.rand(3*space.n_dofs, dtype=torch.float64, device="cuda")
def t(f, n=20):
    f(); torch.cuda.synchronize()
    a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)/n
print("helm nu>0", t(lambda: ops.apply_viscous_helmholtz(space, u, 1500., 1/180, bcs)))
print("helm nu=0", t(lambda: ops.apply_viscous_helmholtz(space, u, 1500., 0.0, bcs)))
ne = mesh.n_elements
td = torch.rand(ne, dtype=torch.float64, device="cuda"); tc = torch.rand(3*ne, dtype=torch.float64, device="cuda")
print("proj full", t(lambda: ops.apply_projection_operator(space, u, td, tc)))
print("proj no tc", t(lambda: ops.apply_projection_operator(space, u, td, None)))
print("proj mass", t(lambda: ops.apply_projection_operator(space, u, None, None)))
print("invmass", t(lambda: ops.inverse_mass_apply(space, u)))
