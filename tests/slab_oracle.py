"""CPU stand-ins of the x-slab device objects for the multi-process gloo
tests (test infrastructure): the numpy oracle applied on a rank's slab
extended by the ghost cell layers it exchanged through the SAME communicator
class the product uses (parallel.TorchComm over gloo), and the rank-local
vector operations of parallel.SlabPCG on torch CPU tensors."""

import numpy as np
import torch

from oracle import dg_oracle as O
from paper_1607_01323_b200.parallel import SlabPartition, slab_of


class OracleSlabLaplace:
    """parallel.SlabLaplace interface (vmult, n_dofs, volume, comm_ops) on the
    CPU.  ``kinds``: oracle boundary kinds per tag of the GLOBAL mesh."""

    def __init__(self, ext, counts, k, per, grading, kinds, rank, world, comm):
        self.counts, self.k, self.comm_ops = counts, k, comm
        self.n = (k + 1) ** 3
        gm = O.build_box_mesh(ext, counts, grading=grading, periodic=per)
        self.gsp = O.DgSpace(gm, k)
        self.gbcs = O.BoundarySpec(kinds).resolve(self.gsp)
        self.volume = float(np.prod([e[1] - e[0] for e in ext]))
        self.part = SlabPartition(counts[0], world, per[0])
        a, b = self.a, self.b = self.part.range(rank)
        self.lo, self.hi = self.part.neighbours(rank)
        self.n_dofs = (b - a) * counts[1] * counts[2] * self.n
        xs = gm.axis_vertices[0]
        ga, gb = a - (self.lo is not None), b + (self.hi is not None)
        hx = np.diff(xs)
        vx = [xs[a] if self.lo is None else xs[a] - hx[(a - 1) % counts[0]]]
        for gx in range(ga, gb):
            vx.append(vx[-1] + hx[gx % counts[0]])
        nxe = gb - ga
        em = O.build_box_mesh(((vx[0], vx[-1]), ext[1], ext[2]), (nxe, counts[1], counts[2]),
                              grading=grading, periodic=(False, per[1], per[2]))
        em.axis_vertices[0] = np.array(vx)
        em.h[:, 0] = np.diff(em.axis_vertices[0])[em.cell_index[0]]
        self.esp = O.DgSpace(em, k)
        # tau of the GLOBAL mesh (ghost cells are interior cells globally)
        gidx = np.array([(ga + i) % counts[0] for i in range(nxe)])
        ix, iy, iz = em.cell_index
        self.esp.tau_e = self.gsp.tau_e[gidx[ix] + counts[0] * (iy + counts[1] * iz)]
        self.esp.tau_if = np.maximum(self.esp.tau_e[self.esp.f_em], self.esp.tau_e[self.esp.f_ep])
        ekinds = dict(kinds)
        ekinds.update({"xmin": O.zero_dirichlet(3), "xmax": O.zero_dirichlet(3)})
        if self.lo is None and not per[0]:
            ekinds["xmin"] = kinds["xmin"]
        if self.hi is None and not per[0]:
            ekinds["xmax"] = kinds["xmax"]
        self.ebcs = O.BoundarySpec(ekinds).resolve(self.esp)
        self.nxe = nxe

    def slab(self, global_field):
        return slab_of(global_field, self.part, self.part_rank(), self.counts, self.n)

    def part_rank(self):
        return [r for r in range(self.part.nranks) if self.part.range(r) == (self.a, self.b)][0]

    def vmult(self, src, dst, tau_scale=1.0):
        nz, ny, n = self.counts[2], self.counts[1], self.n
        loc = src.numpy().reshape(nz, ny, self.b - self.a, n)
        send_lo = torch.from_numpy(np.ascontiguousarray(loc[:, :, 0]).ravel())
        send_hi = torch.from_numpy(np.ascontiguousarray(loc[:, :, -1]).ravel())
        recv_lo, recv_hi = torch.empty_like(send_lo), torch.empty_like(send_hi)
        self.comm_ops.exchange(send_lo, send_hi, recv_lo, recv_hi, self.lo, self.hi)
        layers = []
        if self.lo is not None:
            layers.append(recv_lo.numpy().reshape(nz, ny, 1, n))
        layers.append(loc)
        if self.hi is not None:
            layers.append(recv_hi.numpy().reshape(nz, ny, 1, n))
        ext = np.concatenate(layers, axis=2)
        out = O.apply_pressure_laplace(self.esp, ext.reshape(self.esp.field_shape()), self.ebcs,
                                       tau_scale).reshape(nz, ny, self.nxe, n)
        i0 = 1 if self.lo is not None else 0
        dst.copy_(torch.from_numpy(np.ascontiguousarray(out[:, :, i0:i0 + self.b - self.a]).ravel()))
        return dst


class CpuSlabOps:
    """parallel.DeviceSlabOps on torch CPU tensors (same formulas)."""

    def __init__(self, w, volume):
        self.w, self.vol = w, volume

    def dots(self, p, Lp, out3):
        out3[0] = torch.dot(p, Lp)
        out3[1] = Lp.sum()
        out3[2] = torch.dot(p, self.w)

    def update(self, x, r, p, Lp, scal, project, diag, z, out_rz):
        c = scal[2].item() / self.vol if project else 0.0
        pAp = scal[1].item() - c * scal[3].item() if project else scal[1].item()
        if pAp > 0.0:
            alpha = scal[0].item() / pAp
            x += alpha * p
            r -= alpha * (Lp - c * self.w)
        if diag is not None:
            z.copy_(r / diag)
            out_rz[0] = torch.dot(r, z)

    def pupdate(self, p, z, scal):
        p.copy_(z + (scal[4].item() / scal[0].item()) * p)
        scal[0] = scal[4]

    def dot(self, a, b, out):
        out[0] = torch.dot(a, b)

    def cheb_init(self, r, diag, rc, d, x, theta):
        d.copy_((r / diag) / theta)
        x.copy_(d)
        rc.copy_(r)

    def cheb_step(self, rc, Ld, d_old, d_new, diag, x, a, b):
        rc -= Ld
        d_new.copy_(a * d_old + b * (rc / diag))
        x += d_new
