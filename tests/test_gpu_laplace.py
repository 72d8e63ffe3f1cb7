"""GPU parity of the SIP Laplace path (CUDA kernels via the C ABI).

Bars: relative L2 <= 1e-12 per operator application (BASELINE north star)
against (a) golden vectors produced by the real 2D reference and (b) the
numpy oracle in 3D; identical PCG iteration counts and residual histories
against the reference's own solves.
"""

import numpy as np
import pytest

from tests.golden_setups import KS, SETUPS, load_golden, relerr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1607_01323_b200 import mesh as M  # noqa: E402
from paper_1607_01323_b200 import operators as ops  # noqa: E402
from paper_1607_01323_b200 import solvers as sol  # noqa: E402
from paper_1607_01323_b200.spaces import DgSpace  # noqa: E402
from oracle import dg_oracle as O  # noqa: E402

Z = load_golden()
TOL = 1e-12


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64).ravel(), device="cuda")


def host(t):
    return t.detach().cpu().numpy().ravel()


def gpu_setup(name, k):
    ext, counts, grading, per, kinds = SETUPS[name]
    mesh = M.build_box_mesh(ext, counts, grading=grading, periodic=per)
    space = DgSpace(mesh, k)
    spec = ops.BoundarySpec({t: (ops.DirichletBC(None) if v == "D" else ops.NeumannBC(None, None))
                             for t, v in kinds.items()})
    return space, spec.resolve(space)


@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", KS)
def test_2d_golden_laplace_family(name, k):
    space, bcs = gpu_setup(name, k)
    key = f"{name}_k{k}"
    np.testing.assert_allclose(space.ctx(bcs.kinds).tau(), Z[key + "_tau_e"], rtol=1e-13)
    p = dev(Z[key + "_p"])
    u = dev(Z[key + "_u"])
    checks = {
        "_lap": ops.apply_pressure_laplace(space, p, bcs),
        "_lap75": ops.apply_pressure_laplace(space, p, bcs, tau_scale=7.5),
        "_diag": ops.laplace_diagonal(space, bcs),
        "_diag75": ops.laplace_diagonal(space, bcs, 7.5),
        "_mass": ops.mass_apply(space, u),
        "_invmass": ops.inverse_mass_apply(space, u),
        "_zm": sol.zero_mean_project(space, p),
        "_zmd": sol.zero_mean_project_dual(space, p),
    }
    for suffix, got in checks.items():
        err = relerr(host(got), Z[key + suffix])
        assert err < TOL, (suffix, err)


def test_2d_numpy_reference_layout_roundtrip():
    """numpy inputs in the reference kernel layout (m, ne, m) come back in it."""
    space, bcs = gpu_setup("mixed", 3)
    key = "mixed_k3"
    m, ne = 4, space.mesh.n_elements
    p_em = Z[key + "_p"].reshape(ne, m, m)
    p_ref = np.ascontiguousarray(p_em.transpose(1, 0, 2))
    out = ops.apply_pressure_laplace(space, p_ref, bcs)
    assert out.shape == (m, ne, m)
    got = np.ascontiguousarray(out.transpose(1, 0, 2)).ravel()
    assert relerr(got, Z[key + "_lap"]) < TOL


def oracle_and_gpu_3d(ext, counts, k, periodic, kinds, grading=None):
    om = O.build_box_mesh(ext, counts, grading=grading, periodic=periodic)
    osp = O.DgSpace(om, k)
    ospec = O.BoundarySpec({t: (O.zero_dirichlet(3) if v == "D" else O.zero_neumann(3))
                            for t, v in kinds.items()})
    gm = M.build_box_mesh(ext, counts, grading=grading, periodic=periodic)
    gsp = DgSpace(gm, k)
    gspec = ops.BoundarySpec({t: (ops.DirichletBC(None) if v == "D" else ops.NeumannBC(None, None))
                              for t, v in kinds.items()})
    return osp, ospec.resolve(osp), gsp, gspec.resolve(gsp)


CASES_3D = [
    # extents, counts, periodic, kinds, grading
    (((0, 1), (0, 1), (0, 1)), (3, 4, 5), (True, True, True), {}, None),
    (((0, 1), (0, 2), (0, 1)), (5, 3, 2), (False, False, False),
     {t: "D" for t in O.TAG_NAMES}, None),
    (((0, 2), (-1, 1), (0, 1)), (6, 5, 3), (True, False, True),
     {"ymin": "D", "ymax": "N"}, (0.0, 1.8, 0.0)),
    (((0, 1), (0, 1), (0, 3)), (1, 2, 7), (True, False, False),
     {"ymin": "N", "ymax": "N", "zmin": "D", "zmax": "N"}, (0.0, 0.7, 1.1)),
    (((0, 1), (0, 1), (0, 1)), (9, 1, 2), (False, True, True),
     {"xmin": "N", "xmax": "D"}, (0.5, 0.0, 0.0)),
]


# "auto": the production dispatch (meshes this small run the v4 bricks, the
# multigrid coarse-level rule); "column": DG_LAP_VARIANT=7 forces the z-marching
# column kernels (laplace7 / laplace8) whatever the mesh size
PATHS = {"auto": None, "column": "7"}


@pytest.fixture(params=list(PATHS))
def kernel_path(request, monkeypatch):
    if PATHS[request.param] is None:
        monkeypatch.delenv("DG_LAP_VARIANT", raising=False)
    else:
        monkeypatch.setenv("DG_LAP_VARIANT", PATHS[request.param])
    return request.param


@pytest.mark.parametrize("case", range(len(CASES_3D)))
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7])
def test_3d_laplace_matches_oracle(case, k, kernel_path):
    ext, counts, per, kinds, grading = CASES_3D[case]
    osp, obcs, gsp, gbcs = oracle_and_gpu_3d(ext, counts, k, per, kinds, grading)
    np.testing.assert_allclose(gsp.ctx(gbcs.kinds).tau(), osp.tau_e, rtol=1e-13)
    rng = np.random.default_rng(100 * case + k)
    p = rng.uniform(-1, 1, osp.field_shape())
    for ts in (1.0, 7.5):
        want = O.apply_pressure_laplace(osp, p, obcs, ts).ravel()
        got = host(ops.apply_pressure_laplace(gsp, dev(p), gbcs, ts))
        assert relerr(got, want) < TOL, (ts, relerr(got, want))
    if k <= 4:
        want = O.laplace_diagonal(osp, obcs, 2.0).ravel()
        got = host(ops.laplace_diagonal(gsp, gbcs, 2.0))
        assert relerr(got, want) < TOL
    u = rng.standard_normal(osp.field_shape(3))
    assert relerr(host(ops.mass_apply(gsp, dev(u))), O.mass_apply(osp, u).ravel()) < TOL
    assert relerr(host(ops.inverse_mass_apply(gsp, dev(u))),
                  O.inverse_mass_apply(osp, u).ravel()) < TOL
    assert relerr(host(sol.zero_mean_project(gsp, dev(p))),
                  O.zero_mean_project(osp, p).ravel()) < TOL
    assert relerr(host(sol.zero_mean_project_dual(gsp, dev(p))),
                  O.zero_mean_project_dual(osp, p).ravel()) < TOL


def test_config1_vmult(kernel_path):
    """BASELINE config 1: 8^3 unit cube, Q3, walls, uniform[-1,1] seed 0 --
    both wall kinds (velocity-Dirichlet semantics and the NeumannBC kind
    that exercises the pressure-Dirichlet face branch)."""
    ext = ((0, 1),) * 3
    p = np.random.default_rng(0).uniform(-1, 1, 512 * 64)
    for kind in ("D", "N"):
        kinds = {t: kind for t in O.TAG_NAMES}
        osp, obcs, gsp, gbcs = oracle_and_gpu_3d(ext, (8, 8, 8), 3, (False,) * 3, kinds)
        want = O.apply_pressure_laplace(osp, p.reshape(osp.field_shape()), obcs).ravel()
        got = host(ops.apply_pressure_laplace(gsp, dev(p), gbcs))
        assert relerr(got, want) < TOL


BRICK_CASES = [
    # several full bricks per axis of every kernel's tiling, bench BCs (walls
    # everywhere, velocity-Dirichlet kind), the NeumannBC kind, grading, and
    # partial bricks / partial z-columns
    ((16, 8, 8), (False, False, False), "D", None),
    ((16, 8, 8), (False, False, False), "N", (0.6, 1.2, 0.9)),
    ((12, 10, 9), (True, False, True), "D", (0.0, 1.8, 0.0)),
    ((8, 12, 20), (True, True, False), "N", None),
]


@pytest.mark.parametrize("case", range(len(BRICK_CASES)))
@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_vmult_multibrick_matches_oracle(case, k, kernel_path):
    counts, per, kind, grading = BRICK_CASES[case]
    kinds = {t: kind for t in O.TAG_NAMES}
    ext = ((0, 1), (0, 2), (0, 1))
    osp, obcs, gsp, gbcs = oracle_and_gpu_3d(ext, counts, k, per, kinds, grading)
    p = np.random.default_rng(11 * case + k).uniform(-1, 1, osp.field_shape())
    want = O.apply_pressure_laplace(osp, p, obcs).ravel()
    got = host(ops.apply_pressure_laplace(gsp, dev(p), gbcs))
    assert relerr(got, want) < TOL, relerr(got, want)


@pytest.mark.parametrize("k,nx", [(3, 8), (4, 6)])
def test_pcg_histories_match_reference_2d(k, nx):
    """Fused device PCG vs the reference's own solves (golden): Chebyshev(5,20)
    over Jacobi and plain Jacobi on the pure-Neumann problem (2D analogue of
    config 2): identical iteration counts, residual histories to 1e-10
    (Chebyshev; full history) and 1e-9 (Jacobi; first 60 iterations, see
    SURVEY.md section 7 hard part 4 on summation-order sensitivity)."""
    mesh = M.build_box_mesh(((0, 1), (0, 1)), (nx, nx), periodic=(True, False))
    space = DgSpace(mesh, k)
    bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None),
                            "ymax": ops.DirichletBC(None)}).resolve(space)
    key = f"cg_k{k}_n{nx}"
    diag = ops.laplace_diagonal(space, bcs)
    seed = sol.zero_mean_project(space, dev(Z[key + "_seed"]))
    L = lambda v: ops.apply_pressure_laplace(space, v, bcs)
    lmax, _ = sol.eigen_estimate_via_cg(lambda v: sol.zero_mean_project(space, L(v)),
                                        diag, seed, 20)
    assert abs(lmax - float(Z[key + "_lmax"])) < 1e-11 * lmax
    cfg = sol.ChebyshevConfig(5, 20.0, 1.1 * float(Z[key + "_lmax"]))
    b = dev(Z[key + "_b"])
    for pname, cheb in (("cheb", cfg), ("jac", None)):
        x, st = sol.laplace_pcg(space, bcs, b, project_dual=True, cheb=cheb, diag=diag,
                                rel_tol=1e-10, max_iter=2000)
        assert st.converged
        assert st.iterations == int(Z[f"{key}_{pname}_iters"]), (pname, st.iterations)
        ref = Z[f"{key}_{pname}_hist"]
        n = len(ref) if pname == "cheb" else 60
        np.testing.assert_allclose(np.array(st.history)[:n], ref[:n],
                                   rtol=1e-10 if pname == "cheb" else 1e-9,
                                   atol=1e-13 * ref[0])
        assert relerr(host(x), Z[f"{key}_{pname}_x"]) < 1e-9


def test_generic_pcg_callables_match_fused():
    """The reference-signature pcg(op, prec, b) with device callables gives
    the same iterates as the fused solver."""
    mesh = M.build_box_mesh(((0, 1),) * 3, (4, 4, 4), periodic=(True, False, True))
    space = DgSpace(mesh, 3)
    bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None),
                            "ymax": ops.DirichletBC(None)}).resolve(space)
    diag = ops.laplace_diagonal(space, bcs)
    b = sol.zero_mean_project_dual(space, dev(np.random.default_rng(5).standard_normal(space.n_dofs)))
    L = lambda v: ops.apply_pressure_laplace(space, v, bcs)
    op = lambda v: sol.zero_mean_project_dual(space, L(v))
    cfg = sol.ChebyshevConfig(5, 20.0, 2.3)
    x1, s1 = sol.pcg(op, lambda r: sol.chebyshev_smooth(L, diag, cfg, r), b, rel_tol=1e-10)
    x2, s2 = sol.laplace_pcg(space, bcs, b, project_dual=True, cheb=cfg, diag=diag, rel_tol=1e-10)
    assert s1.iterations == s2.iterations
    # torch (cuBLAS) vs deterministic fixed-order dots: histories agree to
    # 1e-10 of the initial residual (summation-order sensitivity)
    np.testing.assert_allclose(s1.history, s2.history, rtol=1e-7,
                               atol=1e-10 * s1.history[0])
    assert relerr(host(x1), host(x2)) < 1e-9


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_slab_split_equals_full_on_one_gpu(k):
    """x-slab decomposition path (ghost layers + interior/boundary parts) on
    one GPU: slab contexts whose ghost buffers are filled by device copies
    (standing in for the NCCL exchange) reproduce the single-context vmult.
    k = 3..5: face-trace ghost payload (column kernel); k = 2: ghost cells."""
    import ctypes
    from paper_1607_01323_b200 import _lib
    from paper_1607_01323_b200.parallel import SlabPartition, slab_of
    from paper_1607_01323_b200.spaces import DeviceContext
    from paper_1607_01323_b200.operators import ctypes_ptr, _stream
    ext, counts = ((0, 1),) * 3, (8, 4, 3)
    # x grading: the ghost cell's h and tau differ from the owner's (the ghost
    # side coefficients of the split vmult's phase 2)
    for nranks in (2, 3):
        for per, gx in (((False, False, True), 0.0), ((True, False, True), 0.0),
                        ((False, False, True), 0.8)):
            mesh = M.build_box_mesh(ext, counts, periodic=per, grading=(gx, 0.9, 0.0))
            space = DgSpace(mesh, k)
            kinds = {t: ops.NeumannBC(None, None) for t in mesh.boundary_tags()}
            bcs = ops.BoundarySpec(kinds).resolve(space)
            n = space.n_local
            p = np.random.default_rng(7).uniform(-1, 1, space.n_dofs)
            full = host(ops.apply_pressure_laplace(space, dev(p), bcs))
            part = SlabPartition(counts[0], nranks, per[0])
            ctxs, locs, sends, recvs = [], [], [], []
            st = _stream()
            for r in range(nranks):
                c = DeviceContext(mesh, k, bcs.kinds, 0, part.range(r))
                cnt = ctypes.c_int64()
                _lib.call("dg_halo_count", c.handle, ctypes.byref(cnt))
                loc = dev(slab_of(p, part, r, counts, n))
                snd = [torch.empty(cnt.value, dtype=torch.float64, device="cuda") for _ in range(2)]
                rcv = [torch.full((cnt.value,), np.nan, dtype=torch.float64, device="cuda")
                       for _ in range(2)]
                lo, hi = part.neighbours(r)
                _lib.call("dg_halo_attach", c.handle,
                          ctypes_ptr(rcv[0].data_ptr() if lo is not None else 0),
                          ctypes_ptr(rcv[1].data_ptr() if hi is not None else 0))
                _lib.call("dg_halo_pack", c.handle, ctypes_ptr(loc.data_ptr()),
                          ctypes_ptr(snd[0].data_ptr()), ctypes_ptr(snd[1].data_ptr()), st)
                ctxs.append(c); locs.append(loc); sends.append(snd); recvs.append(rcv)
            for r in range(nranks):
                lo, hi = part.neighbours(r)
                if lo is not None:
                    recvs[r][0].copy_(sends[lo][1])
                if hi is not None:
                    recvs[r][1].copy_(sends[hi][0])
            outs, outs2 = [], []
            for r in range(nranks):
                out = torch.full_like(locs[r], np.nan)
                for prt in (1, 2):
                    _lib.call("dg_laplace_vmult_part", ctxs[r].handle,
                              ctypes_ptr(locs[r].data_ptr()), ctypes_ptr(out.data_ptr()),
                              1.0, prt, st)
                outs.append(out.cpu().numpy().reshape(counts[2], counts[1], -1, n))
                if k >= 3:  # traced ghosts: whole slab on zero traces + ghost lifts
                    out2 = torch.full_like(locs[r], np.nan)
                    for phase in (1, 2):
                        _lib.call("dg_laplace_vmult_split", ctxs[r].handle,
                                  ctypes_ptr(locs[r].data_ptr()), ctypes_ptr(out2.data_ptr()),
                                  1.0, phase, st)
                    outs2.append(out2.cpu().numpy().reshape(counts[2], counts[1], -1, n))
            got = np.concatenate(outs, axis=2).ravel()
            assert relerr(got, full) < 1e-14, (nranks, per)
            if outs2:
                got2 = np.concatenate(outs2, axis=2).ravel()
                assert relerr(got2, full) < 1e-14, ("split", nranks, per, relerr(got2, full))


@pytest.mark.parametrize("cells,k", [(64, 4), (40, 3), (40, 5)])
def test_chunk_models_bitwise_equal(cells, k, monkeypatch):
    """The z-chunk length of the column kernels (list-scheduling model: a short
    last chunk per column) only cuts the march differently: the vmult is
    bitwise identical to the one chunked by the older rule (DG_CHUNK_MODEL=0)
    and to one long chunk per column is not required -- chunks re-derive the
    z-neighbour functionals from the same data."""
    mesh = M.build_box_mesh(((0, 1),) * 3, (cells,) * 3, periodic=(False, True, False))
    space = DgSpace(mesh, k)
    bcs = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()}).resolve(space)
    g = torch.Generator(device="cuda").manual_seed(11)
    p = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a = ops.apply_pressure_laplace(space, p, bcs).clone()
    monkeypatch.setenv("DG_CHUNK_MODEL", "0")
    b = ops.apply_pressure_laplace(space, p, bcs).clone()
    monkeypatch.setenv("DG_CHUNK_OLD", "1")
    c = ops.apply_pressure_laplace(space, p, bcs).clone()
    assert torch.equal(a, b) and torch.equal(a, c)


def test_large_periodic_properties():
    """Size-independent properties at 64^3 Q4 (33.5M DoFs): L 1 = 0 on the
    fully periodic box, symmetry <Lp, q> = <p, Lq>, linearity."""
    mesh = M.build_box_mesh(((0, 1),) * 3, (64, 64, 64), periodic=(True, True, True))
    space = DgSpace(mesh, 4)
    bcs = ops.BoundarySpec({}).resolve(space)
    one = torch.ones(space.n_dofs, dtype=torch.float64, device="cuda")
    assert ops.apply_pressure_laplace(space, one, bcs).abs().max().item() < 1e-10
    g = torch.Generator(device="cuda").manual_seed(4)
    p = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    q = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    Lp = ops.apply_pressure_laplace(space, p, bcs)
    Lq = ops.apply_pressure_laplace(space, q, bcs)
    s1, s2 = torch.dot(Lp, q).item(), torch.dot(p, Lq).item()
    assert abs(s1 - s2) <= 1e-11 * abs(s1)
    Lc = ops.apply_pressure_laplace(space, 1.5 * p - 0.25 * q, bcs)
    assert ((Lc - (1.5 * Lp - 0.25 * Lq)).norm() / Lc.norm()).item() < 1e-13


@pytest.mark.parametrize("per", [(False, False, False), (True, True, True), (False, True, True)])
@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_host_buffer_vmult_matches_device(per, k):
    """dg_laplace_vmult_host (chunked H2D / vmult / D2H on three streams) is
    bitwise identical to the device vmult, for several chunk counts."""
    from paper_1607_01323_b200 import operators as ops
    mesh = M.build_box_mesh(((0, 1), (0, 2), (0, 1)), (6, 4, 13), periodic=per)
    space = DgSpace(mesh, k)
    spec = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()})
    bcs = spec.resolve(space)
    x = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda")
    want = ops.apply_pressure_laplace(space, x, bcs).cpu()
    h = x.cpu().pin_memory()
    for chunks in (1, 2, 3, 16):
        ops.HOST_CHUNKS = chunks
        got = ops.apply_pressure_laplace(space, h, bcs)
        assert got.device.type == "cpu" and torch.equal(got, want), chunks
    ops.HOST_CHUNKS = 32


@pytest.mark.parametrize("k", [1, 3, 4, 6])
def test_fused_chebyshev_smooth_matches_generic(k):
    """dg_cheb_step (vmult + Chebyshev update in one kernel) == the
    reference-form chebyshev_smooth with the Laplace callable."""
    from paper_1607_01323_b200 import operators as ops
    mesh = M.build_box_mesh(((0, 1), (0, 2), (0, 1)), (4, 3, 4), periodic=(True, False, True))
    space = DgSpace(mesh, k)
    bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.NeumannBC(None, None)}
                           ).resolve(space)
    diag = ops.laplace_diagonal(space, bcs)
    cfg = sol.ChebyshevConfig(5, 20.0, 2.7)
    b = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda")
    x0 = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda")
    L = lambda v: ops.apply_pressure_laplace(space, v, bcs)
    for xin in (None, x0):
        want = sol.chebyshev_smooth(L, diag, cfg, b, xin)
        got = sol.laplace_chebyshev_smooth(space, bcs, diag, cfg, b, xin)
        assert relerr(got.cpu().numpy(), want.cpu().numpy()) < 1e-13


@pytest.mark.parametrize("k", [3, 4])
def test_column_chebyshev_epilogue(k):
    """The fused Chebyshev step on a mesh of >= 16384 cells equals the
    reference-form chebyshev_smooth with the Laplace callable, partial tiles
    and walls included (36 x 20 x 24 cells, graded y).  Q4: the column
    kernel's cooperative epilogue (laplace8 kEpiCheb, the default there);
    Q3: the v4 bricks (laplace7 kEpiCheb with DG_EPI_COL=1 in the
    environment)."""
    from paper_1607_01323_b200 import operators as ops
    mesh = M.build_box_mesh(((0, 1), (0, 2), (0, 1)), (36, 20, 24), periodic=(True, False, True),
                            grading=(0.0, 1.2, 0.0))
    space = DgSpace(mesh, k)
    bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.NeumannBC(None, None)}
                           ).resolve(space)
    diag = ops.laplace_diagonal(space, bcs)
    cfg = sol.ChebyshevConfig(5, 20.0, 2.7)
    g = torch.Generator(device="cuda").manual_seed(5)
    b = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda", generator=g)
    x0 = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda", generator=g)
    L = lambda v: ops.apply_pressure_laplace(space, v, bcs)
    for xin in (None, x0):
        want = sol.chebyshev_smooth(L, diag, cfg, b, xin)
        got = sol.laplace_chebyshev_smooth(space, bcs, diag, cfg, b, xin)
        assert relerr(got.cpu().numpy(), want.cpu().numpy()) < 1e-13


def test_column_epilogue_pcg_q4():
    """Fused Chebyshev-Jacobi PCG on a Q4 mesh of >= 16384 cells (laplace8
    kEpiDot / kEpiCheb epilogues) against the reference-signature pcg with
    device callables: same iteration count, histories and solution."""
    mesh = M.build_box_mesh(((0, 1), (0, 2), (0, 1)), (36, 20, 24), periodic=(True, False, True),
                            grading=(0.0, 1.2, 0.0))
    space = DgSpace(mesh, 4)
    bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None),
                            "ymax": ops.DirichletBC(None)}).resolve(space)
    diag = ops.laplace_diagonal(space, bcs)
    b = sol.zero_mean_project_dual(space, dev(np.random.default_rng(6).standard_normal(space.n_dofs)))
    L = lambda v: ops.apply_pressure_laplace(space, v, bcs)
    op = lambda v: sol.zero_mean_project_dual(space, L(v))
    cfg = sol.ChebyshevConfig(5, 20.0, 2.8)
    x1, s1 = sol.pcg(op, lambda r: sol.chebyshev_smooth(L, diag, cfg, r), b, rel_tol=1e-8)
    x2, s2 = sol.laplace_pcg(space, bcs, b, project_dual=True, cheb=cfg, diag=diag, rel_tol=1e-8)
    assert s1.converged and s2.converged
    assert s1.iterations == s2.iterations
    np.testing.assert_allclose(s1.history, s2.history, rtol=1e-7, atol=1e-10 * s1.history[0])
    assert relerr(host(x1), host(x2)) < 1e-8
