"""Multi-rank x-slab path on CPU (gloo, world_size 2 and 3).

Exercises the host logic of the N>1 path without a GPU: slab partition,
neighbour ranks (periodic wrap, including the two-rank case where lo == hi),
ghost-layer packing order (the layout dg_halo_pack produces: first/last owned
x-layer, cells ordered (iz, iy)), the send/recv issue-order convention of
parallel.exchange_halos, and the all-reduce of CG partial sums.  The local
operator is the numpy oracle on the slab extended by its ghost layers (tau of
the ghost cells injected from the global mesh); the result must equal the
global operator restricted to the slab.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1607_01323_b200.parallel import (SlabPartition, allreduce_sum, exchange_halos,
                                            slab_of)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, counts, k, periodic_x, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import dg_oracle as O
        ext = ((0.0, 1.0), (0.0, 2.0), (0.0, 1.0))
        per = (periodic_x, False, True)
        grading = (0.0, 0.9, 0.0)
        kinds = {"ymin": O.zero_neumann(3), "ymax": O.zero_dirichlet(3)}
        if not periodic_x:
            kinds.update({"xmin": O.zero_neumann(3), "xmax": O.zero_neumann(3)})
        gm = O.build_box_mesh(ext, counts, grading=grading, periodic=per)
        gsp = O.DgSpace(gm, k)
        gbcs = O.BoundarySpec(kinds).resolve(gsp)
        n = (k + 1) ** 3
        p = np.random.default_rng(3).uniform(-1, 1, gsp.n_local * gm.n_elements)
        full = O.apply_pressure_laplace(gsp, p.reshape(gsp.field_shape()), gbcs).ravel()

        part = SlabPartition(counts[0], world, periodic_x)
        a, b = part.range(rank)
        lo, hi = part.neighbours(rank)
        loc = slab_of(p, part, rank, counts, n).reshape(counts[2], counts[1], b - a, n)
        send_lo = torch.from_numpy(np.ascontiguousarray(loc[:, :, 0]).ravel())
        send_hi = torch.from_numpy(np.ascontiguousarray(loc[:, :, -1]).ravel())
        recv_lo = torch.full_like(send_lo, np.nan)
        recv_hi = torch.full_like(send_hi, np.nan)
        for r in exchange_halos(send_lo, send_hi, recv_lo, recv_hi, lo, hi):
            r.wait()
        # extended slab: [ghost lo] + owned + [ghost hi] along x
        layers = []
        xs = gm.axis_vertices[0]
        xlo, xhi = xs[a], xs[b]
        ga, gb = a, b
        if lo is not None:
            layers.append(recv_lo.numpy().reshape(counts[2], counts[1], 1, n))
            ga = a - 1
        layers.append(loc)
        if hi is not None:
            layers.append(recv_hi.numpy().reshape(counts[2], counts[1], 1, n))
            gb = b + 1
        ext_arr = np.concatenate(layers, axis=2)
        nxe = ext_arr.shape[2]
        # vertex coordinates of the extended slab (ghost cells keep their size)
        hx = np.diff(xs)
        vx = [xlo]
        for gx in range(ga, gb):
            vx.append(vx[-1] + hx[gx % counts[0]])
        em = O.build_box_mesh(((vx[0], vx[-1]), ext[1], ext[2]), (nxe, counts[1], counts[2]),
                              grading=grading, periodic=(False, False, True))
        em.axis_vertices[0] = np.array(vx) - vx[0] + vx[0]
        em.h[:, 0] = np.diff(em.axis_vertices[0])[em.cell_index[0]]
        esp = O.DgSpace(em, k)
        # inject the global tau (ghost cells are not boundary cells globally)
        gidx = np.array([(ga + i) % counts[0] for i in range(nxe)])
        ix, iy, iz = em.cell_index
        gcell = gidx[ix] + counts[0] * (iy + counts[1] * iz)
        esp.tau_e = gsp.tau_e[gcell]
        esp.tau_if = np.maximum(esp.tau_e[esp.f_em], esp.tau_e[esp.f_ep])
        ekinds = dict(kinds)
        ekinds.update({"xmin": O.zero_dirichlet(3), "xmax": O.zero_dirichlet(3)})
        if lo is None and not periodic_x:
            ekinds["xmin"] = kinds["xmin"]
        if hi is None and not periodic_x:
            ekinds["xmax"] = kinds["xmax"]
        ebcs = O.BoundarySpec(ekinds).resolve(esp)
        out = O.apply_pressure_laplace(esp, ext_arr.reshape(esp.field_shape()), ebcs)
        out = out.reshape(counts[2], counts[1], nxe, n)
        i0 = 1 if lo is not None else 0
        mine = out[:, :, i0:i0 + (b - a)].ravel()
        want = slab_of(full, part, rank, counts, n)
        err = np.linalg.norm(mine - want) / np.linalg.norm(want)
        # CG scalar: all-reduced dot of slab pieces == global dot
        part_dot = torch.tensor([float(np.dot(slab_of(p, part, rank, counts, n),
                                              slab_of(full, part, rank, counts, n)))],
                                dtype=torch.float64)
        allreduce_sum(part_dot)
        gdot = float(np.dot(p, full))
        q.put((rank, err, abs(part_dot.item() - gdot) / abs(gdot)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,periodic_x", [(2, False), (2, True), (3, True), (3, False)])
def test_slab_halo_exchange_gloo(world, periodic_x):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    counts, k = (6, 3, 2), 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, counts, k, periodic_x, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, derr in res:
        assert err < 1e-13, (rank, err)
        assert derr < 1e-13, (rank, derr)


def test_partition_and_neighbours():
    part = SlabPartition(128, 8, False)
    assert [part.range(r) for r in range(8)] == [(16 * r, 16 * r + 16) for r in range(8)]
    assert part.neighbours(0) == (None, 1) and part.neighbours(7) == (6, None)
    part = SlabPartition(10, 3, True)
    assert [part.range(r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert part.neighbours(0) == (2, 1) and part.neighbours(2) == (1, 0)
    assert SlabPartition(5, 1, True).neighbours(0) == (None, None)
    with pytest.raises(ValueError):
        SlabPartition(4, 5, False)


def _pcg_worker(rank, world, port, cheb_on, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import dg_oracle as O
        from paper_1607_01323_b200.parallel import SlabPCG, TorchComm
        from tests.slab_oracle import CpuSlabOps, OracleSlabLaplace
        ext, counts, k = ((0.0, 1.0), (0.0, 2.0), (0.0, 1.0)), (6, 3, 2), 2
        per, grading = (True, False, True), (0.0, 0.8, 0.0)
        kinds = {"ymin": O.zero_dirichlet(3), "ymax": O.zero_dirichlet(3)}
        lap = OracleSlabLaplace(ext, counts, k, per, grading, kinds, rank, world, TorchComm())
        gsp, gbcs = lap.gsp, lap.gbcs
        # the pure-Neumann problem of BASELINE config 2, reduced
        L = lambda v: O.apply_pressure_laplace(gsp, v, gbcs)
        diag = O.laplace_diagonal(gsp, gbcs)
        b = O.zero_mean_project_dual(gsp, np.random.default_rng(5).standard_normal(
            gsp.field_shape()))
        cfg = O.chebyshev_from_lanczos(gsp, L, diag, project=O.zero_mean_project) if cheb_on else None
        op = lambda v: O.zero_mean_project_dual(gsp, L(v))
        prec = (lambda r: O.chebyshev_smooth(L, diag, cfg, r)) if cheb_on else (lambda r: r / diag)
        x_ref, st_ref = O.pcg(op, prec, b, rel_tol=1e-10, max_iter=2000)
        T = lambda a: torch.from_numpy(np.ascontiguousarray(lap.slab(np.asarray(a).ravel())))
        w = T(O.dual_weights(gsp))
        solver = SlabPCG(lap, T(diag), cheb=cfg, project_dual=True, ops=CpuSlabOps(w, lap.volume))
        x, st = solver.solve(T(b), rel_tol=1e-10, max_iter=2000)
        xr = lap.slab(x_ref.ravel())
        q.put((rank, st.iterations, st_ref.iterations, st.converged,
               np.array(st.history), np.array(st_ref.history),
               float(np.linalg.norm(x.numpy() - xr) / np.linalg.norm(xr))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cheb_on", [True, False])
def test_sharded_pcg_gloo(world, cheb_on):
    """parallel.SlabPCG over real torch.distributed (gloo) with the oracle as
    the rank-local operator reproduces the oracle's global pcg
    (solvers.py:30-129): identical iteration count and sqrt(r.z) history
    (Chebyshev: full history to 1e-10; Jacobi: first 60 to 1e-9)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_pcg_worker, args=(r, world, port, cheb_on, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, its, its_ref, conv, h, href, xerr in res:
        assert conv and its == its_ref, (rank, its, its_ref)
        m = len(href) if cheb_on else 60
        np.testing.assert_allclose(h[:m], href[:m], rtol=1e-10 if cheb_on else 1e-9,
                                   atol=1e-13 * href[0])
        assert xerr < (1e-10 if cheb_on else 1e-8), (rank, xerr)
