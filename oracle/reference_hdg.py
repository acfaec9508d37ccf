"""CPU ORACLE: direct (non-iterative) HDG solve -- TEST INFRASTRUCTURE ONLY.

Restates the reference module ``ihdg.reference_hdg`` (its
source is absent from /root/reference): assemble the coupled volume + trace
system of Eq. (KHDG) with the trace u_hat as a separate
unknown -- the *unsubstituted* form, SPEC.md:292 ("used only in the oracle")
-- and solve it with a sparse direct method (scipy SuperLU).  Desk scale only
(<= ~2e5 unknowns).  Only ``tests/`` use it: it is the second,
independent oracle of the iteration (the iHDG fixed point must be this HDG
solution, acceptance 2 SPEC.md:504) and the reference
field of the ``vs-direct`` stopping rule.

Formulation (per element K, test v; per face e, test mu in the face space
of degree p, Lagrange at the face GLL nodes; face integrals by (p+2)-point
Gauss quadrature per tangential axis):

  HDGlocal:  -(F(u), grad v)_K + <F_hat(u, u_hat).n, v>_dK + (C u, v)_K = (f, v)_K
  HDGeqn:  <[[F_hat.n]], mu>_e = 0     on interior faces

with the upwind HDG fluxes of the paper:
  transport:  F_hat.n = b.n u + |b.n| (u - u_hat)
  convection-diffusion:  (u_hat n,  sigma.n + b.n u + tau (u - u_hat)),
      tau = (alpha - b.n)/2,  alpha = sqrt(|b.n|^2 + 4)
  shallow water:  (Phi theta.n + sqrt(Phi) (phi - phi_hat),  Phi phi_hat n)
Boundary faces: transport inflow u_hat = g, outflow u_hat = u^-; CD Dirichlet
u_hat = g_D; SW mirror wall phi_hat = phi^- + sqrt(Phi) theta^-.n.
Backward Euler adds (u/dt, v) on the time rows and (u^m/dt, v) to the RHS.

The element quadrature helpers (Basis1D, _Element) are the oracle's own
basis restatement (oracle/ihdg_oracle.py); nothing here shares code with the
iteration's local operators (local_operators), which substitute the trace
formulas instead.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sps
import scipy.sparse.linalg as spla

from .ihdg_oracle import BOUNDARY, Basis1D, OracleProblem, _Element, _kron_axes, structured_neighbors

__all__ = ["DirectHDG", "solve_direct"]

MAX_UNKNOWNS = 400_000


class DirectHDG:
    """Coupled volume + trace system of one steady solve or one backward-Euler step."""

    def __init__(self, prob: OracleProblem, cells, p: int, box=None, periodic=None, dt=None):
        d = prob.dim
        self.prob, self.p, self.dt = prob, p, dt
        self.cells = [int(c) for c in cells]
        self.d = d
        self.periodic = [False] * d if periodic is None else [bool(x) for x in periodic]
        lo = np.zeros(d) if box is None else np.asarray(box[0], float)
        hi = np.ones(d) if box is None else np.asarray(box[1], float)
        self.lo, self.h = lo, (hi - lo) / np.asarray(self.cells, float)
        self.b = Basis1D(p)
        self.el = _Element(self.b, d, self.h)
        self.nel = int(np.prod(self.cells))
        self.nbr = structured_neighbors(self.cells, self.periodic)
        self.m, self.npn = prob.m, self.el.np
        self.nv = self.m * self.npn
        self.nf = (p + 1) ** (d - 1)
        # face basis (Lagrange at the face GLL nodes) at the face Gauss points,
        # tangential axes increasing, the smallest fastest (mesh.py:166-187)
        self.Mu = _kron_axes([self.b.V] * (d - 1)) if d > 1 else np.ones((1, 1))
        self._face_index()
        self.n_faces = self.face_off[-1]
        self.n_unknowns = self.nel * self.nv + self.n_faces * self.nf
        if self.n_unknowns > MAX_UNKNOWNS:
            raise ValueError(f"direct HDG oracle is desk-scale only ({self.n_unknowns} unknowns)")

    # -- face numbering: mesh.py:89-125 order ------------------------------
    def _face_index(self):
        d, c = self.d, self.cells
        self.strides = [int(np.prod(c[:a])) for a in range(d)]
        off = [0]
        for a in range(d):
            ntan = int(np.prod([c[b] for b in range(d) if b != a])) if d > 1 else 1
            planes = c[a] + (0 if self.periodic[a] else 1)
            off.append(off[-1] + planes * ntan)
        self.face_off = off
        e = np.arange(self.nel, dtype=np.int64)
        idx = [(e // self.strides[a]) % c[a] for a in range(d)]
        self.fid = np.zeros((self.nel, 2 * d), dtype=np.int64)
        for a in range(d):
            tl = np.zeros(self.nel, dtype=np.int64)
            mul = 1
            for b in range(d):
                if b != a:
                    tl += idx[b] * mul
                    mul *= c[b]
            ntan = mul
            for s in (0, 1):
                plane = idx[a] + s
                if self.periodic[a]:
                    plane = plane % c[a]
                self.fid[:, 2 * a + s] = off[a] + plane * ntan + tl

    def element_points(self, ref):
        d = self.d
        e = np.arange(self.nel, dtype=np.int64)
        idx = [(e // self.strides[a]) % self.cells[a] for a in range(d)]
        n = len(ref)
        grid = np.indices([n] * d).reshape(d, -1)[::-1]
        pts = np.empty((self.nel, n ** d, d))
        for a in range(d):
            x0 = self.lo[a] + idx[a] * self.h[a]
            pts[:, :, a] = x0[:, None] + 0.5 * (np.asarray(ref)[grid[a]][None, :] + 1.0) * self.h[a]
        return pts

    def _face_node_points(self, K, f):
        """Physical coordinates of the face GLL nodes of local face f of element K."""
        d, n1 = self.d, self.p + 1
        a, s = divmod(f, 2)
        grid = np.indices([n1] * d).reshape(d, -1)[::-1]
        ids = np.flatnonzero(grid[a] == (n1 - 1 if s else 0))
        return self.element_points(self.b.nodes)[K][ids]

    # -- element operators with u_hat free ---------------------------------
    def _element(self):
        """(A0, Cf[f], R): A0 u + sum_f Cf[f] u_hat_f = RHS on every element;
        R: the time-level matrix (u^m rows)."""
        prob, el, d = self.prob, self.el, self.d
        npn, m, nv = self.npn, self.m, self.nv
        sl = [slice(c * npn, (c + 1) * npn) for c in range(m)]
        M = el.mass()
        inv_dt = 0.0 if self.dt is None else 1.0 / self.dt
        A0 = np.zeros((nv, nv))
        R = np.zeros((nv, nv))
        Cf = [np.zeros((nv, self.nf)) for _ in range(2 * d)]
        fm = lambda f, L, Rm: el.fmass(f, L, Rm)   # <R_j, L_i>_f
        if prob.kind == "transport":
            for a in range(d):
                A0 -= prob.beta[a] * el.Q(a)                    # -(u, beta . grad v)
            A0 += (prob.reaction + inv_dt) * M
            R[:] = inv_dt * M
            for f in range(2 * d):
                a, s = divmod(f, 2)
                bn = prob.beta[a] * (1.0 if s else -1.0)
                P = el.Pf[f]
                A0 += (bn + abs(bn)) * fm(f, P, P)              # <b.n u + |b.n| u, v>
                Cf[f] -= abs(bn) * fm(f, P, self.Mu)            # -<|b.n| u_hat, v>
        elif prob.kind == "cd":
            U = d
            for a in range(d):
                A0[sl[a], sl[a]] += M / prob.kappa               # kappa^-1 (sigma, tau)
                A0[sl[a], sl[U]] -= el.Q(a)                      # -(u, div tau)
                A0[sl[U], sl[a]] -= el.Q(a)                      # -(sigma, grad v)
                A0[sl[U], sl[U]] -= prob.beta[a] * el.Q(a)       # -(u, div(beta v))
            A0[sl[U], sl[U]] += (prob.nu + inv_dt) * M
            R[sl[U], sl[U]] = inv_dt * M
            for f in range(2 * d):
                a, s = divmod(f, 2)
                sgn = 1.0 if s else -1.0
                bn = prob.beta[a] * sgn
                tau = 0.5 * (np.sqrt(bn * bn + 4.0) - bn)
                P = el.Pf[f]
                Cf[f][sl[a], :] += sgn * fm(f, P, self.Mu)      # <u_hat n_a, tau_a>
                A0[sl[U], sl[U]] += (bn + tau) * fm(f, P, P)    # <b.n u + tau u, v>
                A0[sl[U], sl[a]] += sgn * fm(f, P, P)           # <sigma.n, v>
                Cf[f][sl[U], :] -= tau * fm(f, P, self.Mu)      # -<tau u_hat, v>
        elif prob.kind == "sw":
            Phi, sP = prob.Phi, np.sqrt(prob.Phi)
            A0[sl[0], sl[0]] += inv_dt * M
            R[sl[0], sl[0]] = inv_dt * M
            for a in range(d):
                th = 1 + a
                A0[sl[0], sl[th]] -= Phi * el.Q(a)               # -(Phi theta, grad phi1)
                A0[sl[th], sl[0]] -= Phi * el.Q(a)               # -(Phi phi, d_a phi2)
                A0[sl[th], sl[th]] += (Phi * inv_dt + prob.gamma * Phi) * M
                R[sl[th], sl[th]] = Phi * inv_dt * M
            A0[sl[1], sl[2]] -= prob.f_cor * Phi * M             # Coriolis (implicit)
            A0[sl[2], sl[1]] += prob.f_cor * Phi * M
            for f in range(2 * d):
                a, s = divmod(f, 2)
                sgn = 1.0 if s else -1.0
                th = 1 + a
                P = el.Pf[f]
                A0[sl[0], sl[th]] += Phi * sgn * fm(f, P, P)    # <Phi theta.n, phi1>
                A0[sl[0], sl[0]] += sP * fm(f, P, P)            # <sqrt(Phi) phi, phi1>
                Cf[f][sl[0], :] -= sP * fm(f, P, self.Mu)       # -<sqrt(Phi) phi_hat, phi1>
                Cf[f][sl[th], :] += Phi * sgn * fm(f, P, self.Mu)  # <Phi phi_hat n_a, phi2>
        else:
            raise ValueError(prob.kind)
        return A0, Cf, R

    def _face_rows(self, f):
        """Flux-jump contributions of one face side: (Fu, Fhat) with
        <F_hat.n, mu> = Fu u_side + Fhat u_hat for the side whose outward face is f."""
        prob, el, d = self.prob, self.el, self.d
        npn, m = self.npn, self.m
        sl = [slice(c * npn, (c + 1) * npn) for c in range(m)]
        a, s = divmod(f, 2)
        sgn = 1.0 if s else -1.0
        P = el.Pf[f]
        Fu = np.zeros((self.nf, self.nv))
        mm = el.fmass(f, self.Mu, P)          # <phi_j, mu_i>
        hh = el.fmass(f, self.Mu, self.Mu)    # <mu_j, mu_i>
        if prob.kind == "transport":
            bn = prob.beta[a] * sgn
            Fu[:, :] = (bn + abs(bn)) * mm
            Fh = -abs(bn) * hh
        elif prob.kind == "cd":
            U = d
            bn = prob.beta[a] * sgn
            tau = 0.5 * (np.sqrt(bn * bn + 4.0) - bn)
            Fu[:, sl[a]] = sgn * mm
            Fu[:, sl[U]] = (bn + tau) * mm
            Fh = -tau * hh
        else:
            Phi, sP = prob.Phi, np.sqrt(prob.Phi)
            Fu[:, sl[1 + a]] = Phi * sgn * mm
            Fu[:, sl[0]] = sP * mm
            Fh = -sP * hh
        return Fu, Fh

    # -- assembly + solve ---------------------------------------------------
    def solve(self, forcing=None, u_prev=None, inflow=None, dirichlet=None):
        """Returns (u (Nel, nv) nodal, u_hat (n_faces, N_f) at the face GLL
        nodes, mesh.py face order).  forcing(x) on the forcing component;
        u_prev: the time level u^m (backward Euler); inflow(x) / dirichlet(x):
        boundary data g at the boundary face nodes (default 0)."""
        prob, d, nv, nf = self.prob, self.d, self.nv, self.nf
        nel = self.nel
        A0, Cf, R = self._element()
        rows, cols, vals = [], [], []

        def add(r0, c0, blk):
            ii, jj = np.nonzero(blk)
            rows.append(r0[:, None] + ii[None, :])
            cols.append(c0[:, None] + jj[None, :])
            vals.append(np.broadcast_to(blk[ii, jj], (len(r0), len(ii))))

        E = np.arange(nel, dtype=np.int64)
        vol0 = E * nv
        add(vol0, vol0, A0)
        hat0 = nel * nv
        for f in range(2 * d):
            add(vol0, hat0 + self.fid[:, f] * nf, Cf[f])
        rhs = np.zeros(self.n_unknowns)
        if forcing is not None:
            pts = self.element_points(self.b.qx)
            fq = np.asarray(forcing(pts.reshape(-1, d)), float).reshape(nel, -1)
            c = prob.forcing_comp
            rhs[(vol0[:, None] + c * self.npn + np.arange(self.npn)[None, :]).ravel()] += \
                ((fq * self.el.W[None, :]) @ self.el.Phi).ravel()
        if u_prev is not None and self.dt is not None:
            up = np.asarray(u_prev, float).reshape(nel, nv)
            rhs[:nel * nv] += (up @ R.T).ravel()
        # face equations: interior = flux jump, boundary = boundary condition
        hh = None
        for a in range(d):
            fo, fn = 2 * a + 1, 2 * a        # owner (normal +e_a) / neighbour side
            Fuo, Fho = self._face_rows(fo)
            Fun, Fhn = self._face_rows(fn)
            nb = self.nbr[:, fo]
            own = np.flatnonzero(nb != BOUNDARY)
            if own.size:
                r0 = hat0 + self.fid[own, fo] * nf
                add(r0, vol0[own], Fuo)
                add(r0, vol0[nb[own]], Fun)
                jump_h = Fho + Fhn
                if prob.kind == "transport" and prob.beta[a] == 0.0:
                    jump_h = -self.el.fmass(fo, self.Mu, self.Mu)   # u_hat unused: pin it
                add(r0, r0, jump_h)
            for s in (0, 1):
                f = 2 * a + s
                bnd = np.flatnonzero(self.nbr[:, f] == BOUNDARY)
                if bnd.size == 0:
                    continue
                sgn = 1.0 if s else -1.0
                r0 = hat0 + self.fid[bnd, f] * nf
                hh = self.el.fmass(f, self.Mu, self.Mu)
                mm = self.el.fmass(f, self.Mu, self.el.Pf[f])
                g = None
                if prob.kind == "transport":
                    bn = prob.beta[a] * sgn
                    if bn < 0:                       # inflow: u_hat = g
                        add(r0, r0, hh)
                        g = inflow
                    else:                            # outflow: u_hat = u^-
                        add(r0, r0, hh)
                        blk = np.zeros((nf, nv))
                        blk[:, :self.npn] = -mm
                        add(r0, vol0[bnd], blk)
                elif prob.kind == "cd":              # Dirichlet: u_hat = g_D
                    add(r0, r0, hh)
                    g = dirichlet
                else:                                # mirror wall
                    add(r0, r0, hh)
                    blk = np.zeros((nf, nv))
                    blk[:, :self.npn] = -mm
                    blk[:, (1 + a) * self.npn:(2 + a) * self.npn] = -np.sqrt(prob.Phi) * sgn * mm
                    add(r0, vol0[bnd], blk)
                if g is not None:
                    gv = np.stack([np.asarray(g(self._face_node_points(int(K), f)), float) for K in bnd])
                    rhs[(r0[:, None] + np.arange(nf)[None, :]).ravel()] += (gv @ hh.T).ravel()
        Amat = sps.csc_matrix((np.concatenate([v.ravel() for v in vals]),
                               (np.concatenate([r.ravel() for r in rows]),
                                np.concatenate([c.ravel() for c in cols]))),
                              shape=(self.n_unknowns, self.n_unknowns))
        x = spla.spsolve(Amat, rhs)
        res = np.linalg.norm(Amat @ x - rhs) / max(np.linalg.norm(rhs), 1e-300)
        if not np.all(np.isfinite(x)) or res > 1e-9:
            raise np.linalg.LinAlgError(f"direct HDG solve failed (relative residual {res:.2e})")
        self.residual = res
        return x[:nel * nv].reshape(nel, nv), x[nel * nv:].reshape(self.n_faces, nf)

    def l2_norm(self, u):
        """||u||_{L2(Omega)} over all components (quadrature, lexicographic sum)."""
        vals = np.asarray(u, float).reshape(self.nel, self.m, self.npn) @ self.el.Phi.T
        return float(np.sqrt(np.add.accumulate(np.einsum("emq,q->e", vals * vals, self.el.W))[-1]))


def solve_direct(prob: OracleProblem, cells, p, box=None, periodic=None, dt=None, **kw):
    """(FieldState data (Nel, m, Np), trace (n_faces, 1, N_f))."""
    D = DirectHDG(prob, cells, p, box=box, periodic=periodic, dt=dt)
    u, t = D.solve(**kw)
    return u.reshape(D.nel, D.m, D.npn), t[:, None, :]
