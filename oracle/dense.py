"""Dense naive-quadrature assembly, DIM in {2, 3} -- TEST INFRASTRUCTURE.

Restates the reference's independent dense oracle (pkg/src/dgins/oracle.py:
15-435: full tensor shape tables, explicit loops over cells and faces,
global dense matrices in element-major order, no sum factorisation) for
2D and 3D Cartesian meshes.  It pins ``dg_oracle``'s sum-factorised 3D
restatement, for which no reference code exists.  Meshes must be tiny
(<= ~27 cells).
"""

import numpy as np

from .dg_oracle import _lax_friedrichs, _face_points, _vol_points


def _kron_all(mats):
    out = mats[0]
    for m in mats[1:]:
        out = np.kron(out, m)
    return out


class DenseOracle:
    def __init__(self, space):
        self.space = space
        self.dim = space.dim
        self.m = space.k + 1
        self.nloc = self.m ** self.dim
        self.ne = space.mesh.n_elements
        self.n_scalar = self.ne * self.nloc
        self.tables = self._build_tables(space.basis)
        self.tables_over = self._build_tables(space.basis_over[0])

    def _pos(self, d):
        """Kronecker factor position of direction d (slowest axis first)."""
        return self.dim - 1 - d

    def _build_tables(self, b):
        dim = self.dim
        val = _kron_all([b.S] * dim)
        grads = []
        for dg in range(dim):
            f = [b.S] * dim
            f[self._pos(dg)] = b.D
            grads.append(_kron_all(f))
        fval, fgrad = {}, {}
        for d in range(dim):
            for s in (0, 1):
                slot = 2 * d + s
                f = [b.S] * dim
                f[self._pos(d)] = b.end_value(s)[None, :]
                fval[slot] = _kron_all(f)
                gl = []
                for dg in range(dim):
                    f = [b.S] * dim
                    if dg == d:
                        f[self._pos(d)] = b.end_deriv(s)[None, :]
                    else:
                        f[self._pos(d)] = b.end_value(s)[None, :]
                        f[self._pos(dg)] = b.D
                    gl.append(_kron_all(f))
                fgrad[slot] = gl
        return {"val": val, "grad": grads, "fval": fval, "fgrad": fgrad}

    def _vol_phys(self, e, geom, t):
        jit = geom.jinvT[:, :, e].reshape(self.dim, self.dim, -1)[..., 0]
        w = np.broadcast_to(geom.jxw[e], geom.jxw.shape[1:]).ravel()
        ph = [sum(jit[a, bb] * t["grad"][bb] for bb in range(self.dim))
              for a in range(self.dim)]
        return t["val"], ph, w

    def _face_phys(self, e, s, geom, t):
        jit = geom.jinvT_f[:, :, e].reshape(self.dim, self.dim, -1)[..., 0]
        T = t["fval"][s]
        ph = [sum(jit[a, bb] * t["fgrad"][s][bb] for bb in range(self.dim))
              for a in range(self.dim)]
        return T, ph

    def _normal(self, geom, s, e):
        return [float(geom.normal[a, s, e].ravel()[0]) for a in range(self.dim)]

    def _sj(self, geom, s, e):
        return np.asarray(geom.sjxw[s, e]).ravel()

    def _sd(self, e):
        return np.arange(e * self.nloc, (e + 1) * self.nloc)

    def _vd(self, e):
        s = self._sd(e)
        return np.concatenate([c * self.n_scalar + s for c in range(self.dim)])

    def mass_matrix(self, ncomp=1):
        g = self.space.geom
        A = np.zeros((self.n_scalar, self.n_scalar))
        for e in range(self.ne):
            val, _, w = self._vol_phys(e, g, self.tables)
            A[np.ix_(self._sd(e), self._sd(e))] = val.T @ (w[:, None] * val)
        if ncomp == 1:
            return A
        return np.kron(np.eye(ncomp), A)

    def laplace_matrix(self, bcs, tau_scale=1.0):
        """oracle.py:95-130."""
        sp, g, dim = self.space, self.space.geom, self.dim
        A = np.zeros((self.n_scalar, self.n_scalar))
        for e in range(self.ne):
            _, ph, w = self._vol_phys(e, g, self.tables)
            A[np.ix_(self._sd(e), self._sd(e))] += sum(
                p.T @ (w[:, None] * p) for p in ph)
        f = sp.mesh.interior
        for i in range(f.n):
            em, sm, ep, spp = f.em[i], f.sm[i], f.ep[i], f.sp[i]
            Tm, pm = self._face_phys(em, sm, g, self.tables)
            Tp, pp = self._face_phys(ep, spp, g, self.tables)
            n = self._normal(g, sm, em)
            w = self._sj(g, sm, em)
            tau = tau_scale * sp.tau_if[i]
            avg = 0.5 * np.concatenate([sum(pm[a] * n[a] for a in range(dim)),
                                        sum(pp[a] * n[a] for a in range(dim))],
                                       axis=1)
            jmp = np.concatenate([Tm, -Tp], axis=1)
            blk = (-avg.T @ (w[:, None] * jmp) - jmp.T @ (w[:, None] * avg)
                   + tau * jmp.T @ (w[:, None] * jmp))
            dofs = np.concatenate([self._sd(em), self._sd(ep)])
            A[np.ix_(dofs, dofs)] += blk
        for eb, sb, _ in bcs.neumann:
            for e, s in zip(eb, sb):
                T, ph = self._face_phys(e, s, g, self.tables)
                n = self._normal(g, s, e)
                w = self._sj(g, s, e)
                Gn = sum(ph[a] * n[a] for a in range(dim))
                tau = tau_scale * sp.tau_e[e]
                blk = (-Gn.T @ (w[:, None] * T) - T.T @ (w[:, None] * Gn)
                       + 2.0 * tau * T.T @ (w[:, None] * T))
                A[np.ix_(self._sd(e), self._sd(e))] += blk
        return A

    def helmholtz_matrix(self, bcs, gamma0_dt, nu):
        """oracle.py:132-213, strain form in DIM dimensions."""
        sp, g, dim = self.space, self.space.geom, self.dim
        nsc = self.nloc
        A = gamma0_dt * self.mass_matrix(ncomp=dim)
        if nu == 0.0:
            return A

        def comp_block(tab_list):
            """rows = points, columns = [u_0 | ... | u_dim-1] local dofs."""
            return np.concatenate(tab_list, axis=1)

        for e in range(self.ne):
            _, ph, w = self._vol_phys(e, g, self.tables)
            z = np.zeros_like(ph[0])
            blk = 0.0
            for a in range(dim):
                for bb in range(dim):
                    # eps_ab(u) = 0.5 (d_b u_a + d_a u_b)
                    cols = [z] * dim
                    cols = list(cols)
                    cols[a] = cols[a] + 0.5 * ph[bb]
                    cols[bb] = cols[bb] + 0.5 * ph[a]
                    E = comp_block(cols)
                    blk = blk + 2.0 * nu * E.T @ (w[:, None] * E)
            A[np.ix_(self._vd(e), self._vd(e))] += blk

        def viscn(ph, n):
            """rows of (2 nu eps(u) . n)_a over [u_0..u_dim-1] columns."""
            rows = []
            for a in range(dim):
                cols = [np.zeros_like(ph[0]) for _ in range(dim)]
                for bb in range(dim):
                    cols[a] = cols[a] + nu * ph[bb] * n[bb]
                    cols[bb] = cols[bb] + nu * ph[a] * n[bb]
                rows.append(comp_block(cols))
            return rows

        def valrows(T):
            z = np.zeros_like(T)
            return [comp_block([T if c == a else z for c in range(dim)])
                    for a in range(dim)]

        f = sp.mesh.interior
        for i in range(f.n):
            em, sm, ep, spp = f.em[i], f.sm[i], f.ep[i], f.sp[i]
            Tm, pm = self._face_phys(em, sm, g, self.tables)
            Tp, pp = self._face_phys(ep, spp, g, self.tables)
            n = self._normal(g, sm, em)
            w = self._sj(g, sm, em)
            tau = sp.tau_if[i] * nu
            Vm, Vp = valrows(Tm), valrows(Tp)
            Gm, Gp = viscn(pm, n), viscn(pp, n)
            dofs = np.concatenate([self._vd(em), self._vd(ep)])
            blk = np.zeros((len(dofs), len(dofs)))
            for a in range(dim):
                avg = 0.5 * np.concatenate([Gm[a], Gp[a]], axis=1)
                jmp = np.concatenate([Vm[a], -Vp[a]], axis=1)
                blk += (-avg.T @ (w[:, None] * jmp) - jmp.T @ (w[:, None] * avg)
                        + tau * jmp.T @ (w[:, None] * jmp))
            A[np.ix_(dofs, dofs)] += blk
        for eb, sb, _ in bcs.dirichlet:
            for e, s in zip(eb, sb):
                T, ph = self._face_phys(e, s, g, self.tables)
                n = self._normal(g, s, e)
                w = self._sj(g, s, e)
                tau = sp.tau_e[e] * nu
                V, G = valrows(T), viscn(ph, n)
                blk = 0.0
                for a in range(dim):
                    blk = blk + (-G[a].T @ (w[:, None] * V[a])
                                 - V[a].T @ (w[:, None] * G[a])
                                 + 2.0 * tau * V[a].T @ (w[:, None] * V[a]))
                A[np.ix_(self._vd(e), self._vd(e))] += blk
        del nsc
        return A

    def projection_matrix(self, tau_d_e=None, tau_c_f=None):
        """oracle.py:215-242."""
        sp, g, dim = self.space, self.space.geom, self.dim
        A = self.mass_matrix(ncomp=dim)
        if tau_d_e is not None:
            for e in range(self.ne):
                _, ph, w = self._vol_phys(e, g, self.tables)
                div = np.concatenate(ph, axis=1)
                A[np.ix_(self._vd(e), self._vd(e))] += \
                    tau_d_e[e] * div.T @ (w[:, None] * div)
        if tau_c_f is not None:
            f = sp.mesh.interior
            for i in range(f.n):
                em, sm, ep, spp = f.em[i], f.sm[i], f.ep[i], f.sp[i]
                Tm, _ = self._face_phys(em, sm, g, self.tables)
                Tp, _ = self._face_phys(ep, spp, g, self.tables)
                w = self._sj(g, sm, em)
                dofs = np.concatenate([self._vd(em), self._vd(ep)])
                c = Tm.shape[1]
                blk = np.zeros((2 * dim * c, 2 * dim * c))
                for comp in range(dim):
                    J = np.zeros((len(w), 2 * dim * c))
                    J[:, comp * c:(comp + 1) * c] = Tm
                    J[:, (dim + comp) * c:(dim + comp + 1) * c] = -Tp
                    blk += tau_c_f[i] * J.T @ (w[:, None] * J)
                A[np.ix_(dofs, dofs)] += blk
        return A

    def _boundary_faces(self, bcs):
        for groups in (bcs.dirichlet, bcs.neumann):
            for eb, sb, _ in groups:
                yield from zip(eb, sb)

    def divergence_form_matrix(self, bcs, scale, form):
        """a(q, u), rows pressure / columns velocity (oracle.py:244-295);
        'standard' or 'weak' (central flux, interior trace on boundaries)."""
        sp, g, dim = self.space, self.space.geom, self.dim
        A = np.zeros((self.n_scalar, dim * self.n_scalar))
        t = self.tables
        for e in range(self.ne):
            val, ph, w = self._vol_phys(e, g, t)
            if form == "standard":
                blk = np.concatenate([-scale * val.T @ (w[:, None] * ph[a])
                                      for a in range(dim)], axis=1)
            else:
                blk = np.concatenate([scale * ph[a].T @ (w[:, None] * val)
                                      for a in range(dim)], axis=1)
            A[np.ix_(self._sd(e), self._vd(e))] += blk
        if form == "standard":
            return A
        f = sp.mesh.interior
        for i in range(f.n):
            em, sm, ep, spp = f.em[i], f.sm[i], f.ep[i], f.sp[i]
            Tm, _ = self._face_phys(em, sm, g, t)
            Tp, _ = self._face_phys(ep, spp, g, t)
            n = self._normal(g, sm, em)
            w = self._sj(g, sm, em)
            # {u}.n^- over columns [u_a^- ..., u_a^+ ...]
            Un = np.concatenate([0.5 * Tm * n[a] for a in range(dim)]
                                + [0.5 * Tp * n[a] for a in range(dim)], axis=1)
            cols = np.concatenate([self._vd(em), self._vd(ep)])
            A[np.ix_(self._sd(em), cols)] += -scale * Tm.T @ (w[:, None] * Un)
            A[np.ix_(self._sd(ep), cols)] += scale * Tp.T @ (w[:, None] * Un)
        for e, s in self._boundary_faces(bcs):
            T, _ = self._face_phys(e, s, g, t)
            n = self._normal(g, s, e)
            w = self._sj(g, s, e)
            Un = np.concatenate([T * n[a] for a in range(dim)], axis=1)
            A[np.ix_(self._sd(e), self._vd(e))] += -scale * T.T @ (w[:, None] * Un)
        return A

    def pressure_gradient_matrix(self, bcs, scale, form):
        """b(v, p), rows velocity / columns pressure (oracle.py:297-348)."""
        sp, g, dim = self.space, self.space.geom, self.dim
        A = np.zeros((dim * self.n_scalar, self.n_scalar))
        t = self.tables
        for e in range(self.ne):
            val, ph, w = self._vol_phys(e, g, t)
            if form == "standard":
                blk = np.concatenate([-scale * val.T @ (w[:, None] * ph[a])
                                      for a in range(dim)], axis=0)
            else:
                blk = np.concatenate([scale * ph[a].T @ (w[:, None] * val)
                                      for a in range(dim)], axis=0)
            A[np.ix_(self._vd(e), self._sd(e))] += blk
        if form == "standard":
            return A
        f = sp.mesh.interior
        for i in range(f.n):
            em, sm, ep, spp = f.em[i], f.sm[i], f.ep[i], f.sp[i]
            Tm, _ = self._face_phys(em, sm, g, t)
            Tp, _ = self._face_phys(ep, spp, g, t)
            n = self._normal(g, sm, em)
            w = self._sj(g, sm, em)
            cols = np.concatenate([self._sd(em), self._sd(ep)])
            avg = 0.5 * np.concatenate([Tm, Tp], axis=1)
            A[np.ix_(self._vd(em), cols)] += np.concatenate(
                [-scale * (Tm * n[a]).T @ (w[:, None] * avg) for a in range(dim)], axis=0)
            A[np.ix_(self._vd(ep), cols)] += np.concatenate(
                [scale * (Tp * n[a]).T @ (w[:, None] * avg) for a in range(dim)], axis=0)
        for e, s in self._boundary_faces(bcs):
            T, _ = self._face_phys(e, s, g, t)
            n = self._normal(g, s, e)
            w = self._sj(g, s, e)
            A[np.ix_(self._vd(e), self._sd(e))] += np.concatenate(
                [-scale * (T * n[a]).T @ (w[:, None] * T) for a in range(dim)], axis=0)
        return A

    def convective_residual(self, bcs, history_flat, betas, times, t_np1,
                            body_force=None):
        """oracle.py:350-426."""
        sp, dim = self.space, self.dim
        bo, go = sp.basis_over
        t = self.tables_over
        out = np.zeros(dim * self.n_scalar)
        ns = self.n_scalar

        def comp(uflat, c, e):
            return uflat[c * ns + self._sd(e)]

        for beta, uflat, ti in zip(betas, history_flat, times):
            for e in range(self.ne):
                val, ph, w = self._vol_phys(e, go, t)
                v = [val @ comp(uflat, c, e) for c in range(dim)]
                for a in range(dim):
                    r = sum(ph[bb].T @ (w * v[a] * v[bb]) for bb in range(dim))
                    out[a * ns + self._sd(e)] += beta * r
            f = sp.mesh.interior
            for i in range(f.n):
                em, sm, ep, spp = f.em[i], f.sm[i], f.ep[i], f.sp[i]
                Tm, _ = self._face_phys(em, sm, go, t)
                Tp, _ = self._face_phys(ep, spp, go, t)
                n = self._normal(go, sm, em)
                w = self._sj(go, sm, em)
                um = [Tm @ comp(uflat, c, em) for c in range(dim)]
                up = [Tp @ comp(uflat, c, ep) for c in range(dim)]
                F = _lax_friedrichs(um, up, n)
                for a in range(dim):
                    out[a * ns + self._sd(em)] += -beta * Tm.T @ (w * F[a])
                    out[a * ns + self._sd(ep)] += beta * Tp.T @ (w * F[a])
            for eb, sb, bc in bcs.dirichlet:
                xb = _face_points(sp, go, bo, eb, sb)
                for j, (e, s) in enumerate(zip(eb, sb)):
                    T, _ = self._face_phys(e, s, go, t)
                    n = self._normal(go, s, e)
                    w = self._sj(go, s, e)
                    gu = bc.g(xb[:, j:j + 1], ti)[:, 0].reshape(dim, -1)
                    ub = [T @ comp(uflat, c, e) for c in range(dim)]
                    F = _lax_friedrichs(ub, [2 * gu[a] - ub[a] for a in range(dim)], n)
                    for a in range(dim):
                        out[a * ns + self._sd(e)] += -beta * T.T @ (w * F[a])
            for eb, sb, _ in bcs.neumann:
                for e, s in zip(eb, sb):
                    T, _ = self._face_phys(e, s, go, t)
                    n = self._normal(go, s, e)
                    w = self._sj(go, s, e)
                    ub = [T @ comp(uflat, c, e) for c in range(dim)]
                    un = sum(ub[a] * n[a] for a in range(dim))
                    for a in range(dim):
                        out[a * ns + self._sd(e)] += -beta * T.T @ (w * ub[a] * un)
        if body_force is not None:
            xq = _vol_points(sp, bo)
            for e in range(self.ne):
                val, _, w = self._vol_phys(e, go, t)
                x = xq[:, e].reshape(dim, -1)
                fv = body_force(x, t_np1)
                for a in range(dim):
                    out[a * ns + self._sd(e)] += val.T @ (w * fv[a])
        return out
