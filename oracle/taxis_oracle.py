"""TEST INFRASTRUCTURE ONLY: numpy restatement of the reference DG
operator (the B200 hot path), its SSP-RK3 composition and the SDIRK +
Jacobian-free Newton-GMRES stepper.

Not part of the product: the CUDA path in ``paper_1403_1157_b200`` never
imports this module.  It is the checker in ``tests/`` and the timed CPU
reference arm in ``bench.py``.

It follows the reference's *operation sequence* (full reference
gradients of every species at every quadrature point, diffusion through
the quadrature, the lifting as the (F x F) face-mass product, full
physical gradient averages in the LLF flux), not the reformulated
sequence of the CUDA kernels, so agreement between the two is a real
check.  Setup inputs (mesh arrays, basis and quadrature tables) come
from the product's host-side setup modules, which are themselves pinned
to the reference by ``tests/test_setup_golden.py``; this operator is
pinned to the reference's own outputs by ``tests/test_oracle_golden.py``.

Reference citations are ``pkg/src/taxisdg/<file>:<line>``.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from paper_1403_1157_b200.fespace import face_reference_points
from paper_1403_1157_b200.fields import bump_field  # noqa: F401 (re-export)
from paper_1403_1157_b200.mesh import BoundaryTag, is_gamma1
from paper_1403_1157_b200.model import (MODEL_DIFFUSION, MODEL_PLAQUE,
                                        MODEL_REDUCED)
from paper_1403_1157_b200.quadrature import face_rule, volume_rule

__all__ = ["OracleOperator", "ssprk3", "sdirk_integrate", "bump_field"]

_REF_FACE = {2: 1.0, 3: 0.5}       # operator.py:74


# ----------------------------------------------------------------- physics


def _chi(x, y, a, b):
    """a x / (max(y,0) + b)   (model.py:53-55)."""
    return a * x / (np.maximum(y, 0.0) + b)


def _step(s, eps):
    """Heaviside, logistic when eps > 0   (model.py:58-62)."""
    if eps == 0.0:
        return np.where(s > 0.0, 1.0, 0.0)
    return 1.0 / (1.0 + np.exp(np.clip(-s / eps, -60.0, 60.0)))


class _PlaquePhysics:
    """PlaqueModel pointwise terms (model.py:143-209)."""

    def __init__(self, p):
        self.p = p
        self.A = np.array([p.mu1, p.mu2, p.mu3, p.nu1, p.nu2, p.nu3])

    def flux(self, u, g):                       # model.py:147-157
        p = self.p
        F = np.zeros(u.shape + (g.shape[-1],))
        F[..., 0, :] = (_chi(u[..., 0], u[..., 3], p.chi11_a, p.chi11_b)[..., None]
                        * g[..., 3, :]
                        + _chi(u[..., 0], u[..., 5], p.chi13_a, p.chi13_b)[..., None]
                        * g[..., 5, :])
        F[..., 1, :] = (_chi(u[..., 1], u[..., 3], p.chi21_a, p.chi21_b)[..., None]
                        * g[..., 3, :]
                        - _chi(u[..., 1], u[..., 0], p.chi2n_a, p.chi2n_b)[..., None]
                        * g[..., 0, :])
        return F

    def source(self, u):                        # model.py:159-170
        p = self.p
        n1, n2, n3, c1, c2 = (u[..., i] for i in range(5))
        S = np.empty_like(u)
        S[..., 0] = -p.d1 * n1
        S[..., 1] = -p.d2 * n2
        S[..., 2] = p.d1 * n1 + p.d2 * n2 - p.gamma * n1
        S[..., 3] = -p.alpha1 * n1 * c1 - p.alpha2 * n2 * c1 + p.f1_const * n3
        S[..., 4] = -p.k_ox * c2
        S[..., 5] = p.k_ox * c2
        return S

    def speed(self, uin, uout, g, n):           # model.py:172-192
        p = self.p
        lam = np.zeros(uin.shape[:-1])
        for u in (uin, uout):
            v0 = ((p.chi11_a / (np.maximum(u[..., 3], 0.0) + p.chi11_b))[..., None]
                  * g[..., 3, :]
                  + (p.chi13_a / (np.maximum(u[..., 5], 0.0) + p.chi13_b))[..., None]
                  * g[..., 5, :])
            v1 = ((p.chi21_a / (np.maximum(u[..., 3], 0.0) + p.chi21_b))[..., None]
                  * g[..., 3, :]
                  - (p.chi2n_a / (np.maximum(u[..., 0], 0.0) + p.chi2n_b))[..., None]
                  * g[..., 0, :])
            vn = np.maximum(np.abs((v0 * n).sum(-1)), np.abs((v1 * n).sum(-1)))
            lam = np.maximum(lam, vn)           # other species move with v = 0
        return lam

    def wall(self, tag, u):                     # model.py:194-209
        p = self.p
        q = np.zeros_like(u)
        c1 = u[..., 3]
        if is_gamma1(tag):
            q[..., 0] = -p.mu1 * p.beta1 * _step(c1 - p.c1_star, p.eps_h)
        if tag == BoundaryTag.GAMMA1_IN:
            q[..., 4] = -p.nu2 * p.sigma
        if tag == BoundaryTag.GAMMA2:
            q[..., 1] = -p.mu2 * p.beta2 * _step(c1 - p.c1_starstar, p.eps_h)
        return q


class _ReducedPhysics:
    """ReducedModel (model.py:212-264): species n1, n3, c1."""

    def __init__(self, p):
        self.p = p
        self.A = np.array([p.mu1, p.mu3, p.nu1])

    def flux(self, u, g):
        p = self.p
        F = np.zeros(u.shape + (g.shape[-1],))
        F[..., 0, :] = _chi(u[..., 0], u[..., 2], p.chi11_a,
                            p.chi11_b)[..., None] * g[..., 2, :]
        return F

    def source(self, u):
        p = self.p
        S = np.empty_like(u)
        S[..., 0] = 0.0
        S[..., 1] = p.d1 * u[..., 0] - p.gamma * u[..., 0]
        S[..., 2] = -p.alpha1 * u[..., 0] * u[..., 2] + p.f1_const * u[..., 1]
        return S

    def speed(self, uin, uout, g, n):
        p = self.p
        gn = np.abs((g[..., 2, :] * n).sum(-1))
        lam = np.zeros(uin.shape[:-1])
        for u in (uin, uout):
            lam = np.maximum(lam, gn * p.chi11_a / (np.maximum(u[..., 2], 0.0)
                                                    + p.chi11_b))
        return lam

    def wall(self, tag, u):
        p = self.p
        q = np.zeros_like(u)
        if is_gamma1(tag):
            q[..., 0] = -p.mu1 * p.beta1 * _step(u[..., 2] - p.c1_star, p.eps_h)
        return q


class _DiffusionPhysics:
    """Pure diffusion test models (reference tests/oracles.py:192-220)."""

    def __init__(self, model):
        self.A = model.diffusivity()
        self.dirichlet = model.dirichlet

    def source(self, u):
        return np.zeros_like(u)

    def wall(self, tag, u):
        return np.zeros_like(u)


def _physics(model):
    if model.model_id == MODEL_PLAQUE:
        return _PlaquePhysics(model.params), True
    if model.model_id == MODEL_REDUCED:
        return _ReducedPhysics(model.params), True
    if model.model_id == MODEL_DIFFUSION:
        return _DiffusionPhysics(model), False
    raise ValueError("unknown model")


# ---------------------------------------------------------------- operator


class OracleOperator:
    """CPU restatement of ``DiscreteOperator`` (operator.py:77-458).

    ``nthreads`` > 1 splits the elements by recursive coordinate bisection
    like the reference (mesh.py:432-456); each worker
    assembles the volume terms of its elements and every term of the
    faces whose inside element it owns into a private buffer, merged in
    part order (the reference's owner-computes scheme,
    operator.py:253-284).
    """

    def __init__(self, space, model, scheme, nthreads: int = 1,
                 vol_degree=None, face_degree=None, global_ids=None):
        if model.n_species != space.n_species:
            raise ValueError("species count mismatch")
        self.space, self.model, self.scheme = space, model, scheme
        mesh = self.mesh = space.mesh
        d, k = mesh.dim, space.order
        self.phys, self.conv = _physics(model)
        self.A = np.asarray(self.phys.A, dtype=float)
        self.chi_e = {2: 1.5, 3: 2.0}[d]                      # flux.py:87-89
        self.adj = -1.0 if scheme.name == "bo" else 1.0       # flux.py:79-80
        self.eta = scheme.ip_eta0 * max(k, 1) ** 2            # operator.py:104
        vr = volume_rule(d, 3 * k + 1 if vol_degree is None else vol_degree)
        fr = face_rule(d, 3 * k + 2 if face_degree is None else face_degree)
        self.wv, self.wf = vr.weights, fr.weights
        basis = space.basis
        self.Phi = basis.eval(vr.points)                      # (Q, nb)
        self.Gv = basis.grad(vr.points)                       # (Q, nb, d)
        self.tab = {}
        for lf in range(d + 1):
            for pm in range(2 if d == 2 else 6):
                xi = face_reference_points(d, lf, pm, fr.points)
                B = basis.eval(xi)
                self.tab[lf, pm] = (B, basis.grad(xi),
                                    (B @ B.T) * self.wf[None, :])
        nb = basis.size
        Q = len(self.wv)
        # flattened layouts so the contractions are batched matmuls
        self._GvT = self.Gv.transpose(1, 0, 2).reshape(nb, Q * d)
        self._GvW = (self.wv[:, None, None] * self.Gv).transpose(0, 2, 1) \
            .reshape(Q * d, nb)
        self._PhiW = self.wv[:, None] * self.Phi
        self._GfT = {key: G.transpose(1, 0, 2).reshape(nb, -1)
                     for key, (B, G, P) in self.tab.items()}
        self._GfD = {key: G.transpose(2, 0, 1).reshape(d, -1)
                     for key, (B, G, P) in self.tab.items()}
        _, self.detJ, self.Jinv = mesh.jacobians()
        self.nthreads = max(1, int(nthreads))
        # K- ties break by GLOBAL element id (slab-local meshes renumber)
        self.gid = (np.arange(mesh.n_elements) if global_ids is None
                    else np.asarray(global_ids))
        self._groups()

    def _groups(self):
        """Faces batched by (lf_in, pm_in, lf_out, pm_out) or
        (lf, pm, tag) (operator.py:147-206)."""
        m = self.mesh
        fe = m.face_elems
        fl = m.face_local.astype(np.int64)
        fp = m.face_perm.astype(np.int64)
        interior = fe[:, 1] >= 0
        P = self.nthreads
        ne = m.n_elements
        # the reference's partition: recursive coordinate bisection of the
        # element centroids (mesh.py:432-456), one part per worker
        part_of = m.partition(P) if P > 1 else np.zeros(ne, dtype=np.int64)
        self.parts = [np.flatnonzero(part_of == p) for p in range(P)]
        owner = part_of[fe[:, 0]]
        key = np.where(interior,
                       ((fl[:, 0] * 8 + fp[:, 0]) * 8 + fl[:, 1]) * 8 + fp[:, 1],
                       100000 + (fl[:, 0] * 8 + fp[:, 0]) * 8
                       + m.face_tags.astype(np.int64))
        self.groups = []
        for kv in np.unique(key):
            fids_all = np.flatnonzero(key == kv)
            for p in range(P):
                fids = fids_all[owner[fids_all] == p]
                if len(fids) == 0:
                    continue
                g = {"p": p, "interior": bool(interior[fids[0]]),
                     "ein": fe[fids, 0], "eout": fe[fids, 1],
                     "lin": int(fl[fids[0], 0]), "pin": int(fp[fids[0], 0]),
                     "lout": int(fl[fids[0], 1]), "pout": int(fp[fids[0], 1]),
                     "n": m.face_normals[fids], "tag": int(m.face_tags[fids[0]]),
                     "sfac": m.face_measures[fids] / _REF_FACE[m.dim]}
                h = m.diameters[g["ein"]].copy()
                if g["interior"]:
                    h = np.minimum(h, m.diameters[g["eout"]])
                    vi, vo = m.volumes[g["ein"]], m.volumes[g["eout"]]
                    gi, go = self.gid[g["ein"]], self.gid[g["eout"]]
                    g["minus_in"] = ~((vo < vi) | ((vo == vi) & (go < gi)))
                g["h"] = h
                self.groups.append(g)

    # -- pieces ------------------------------------------------------------

    def _volume(self, U, E, out):                 # operator.py:292-324
        c = U[E]
        ne, S, nb = c.shape
        Q, d = self.Gv.shape[0], self.Gv.shape[2]
        u = np.matmul(self.Phi, c.transpose(0, 2, 1))               # (e,q,s)
        gref = np.matmul(c, self._GvT).reshape(ne, S * Q, d)        # (e,s*q,a)
        Jinv = self.Jinv[E]
        gphys = np.matmul(gref, Jinv)                               # gref @ Jinv
        Ssrc = self.phys.source(u)
        sig = -self.A[None, :, None] * gphys.reshape(ne, S, Q * d)
        if self.conv:
            gp = gphys.reshape(ne, S, Q, d).transpose(0, 2, 1, 3)   # (e,q,s,d)
            F = self.phys.flux(u, gp).transpose(0, 2, 1, 3)
            sig = sig + F.reshape(ne, S, Q * d)
        sref = np.matmul(sig.reshape(ne, S * Q, d),
                         np.swapaxes(Jinv, 1, 2))                   # sig @ Jinv^T
        r = np.matmul(sref.reshape(ne, S, Q * d), self._GvW)
        r += np.matmul(Ssrc.transpose(0, 2, 1), self._PhiW)
        out[E] += self.detJ[E][:, None, None] * r

    def _trace(self, U, elems, lf, pm):            # operator.py:326-334
        B, G, _ = self.tab[lf, pm]
        c = U[elems]
        nF, S, nb = c.shape
        F, d = G.shape[0], G.shape[2]
        return (np.matmul(B, c.transpose(0, 2, 1)),                          # (f,q,s)
                np.matmul(c, self._GfT[lf, pm]).reshape(nF, S, F, d))        # (f,s,q,a)

    def _faces(self, U, g, out):                   # operator.py:359-434
        A = self.A
        name = self.scheme.name
        Bi, Gi, Pi = self.tab[g["lin"], g["pin"]]
        ein = g["ein"]
        n = g["n"]
        uin, grin = self._trace(U, ein, g["lin"], g["pin"])
        nF, S, F, d = grin.shape
        jin = np.matmul(self.Jinv[ein], n[:, :, None])                      # (f,a,1)
        gnin = np.matmul(grin.reshape(nF, S * F, d), jin).reshape(nF, S, F)
        if g["interior"]:
            eout = g["eout"]
            Bo, Go, Po = self.tab[g["lout"], g["pout"]]
            uout, grout = self._trace(U, eout, g["lout"], g["pout"])
            jout = np.matmul(self.Jinv[eout], n[:, :, None])
            gnout = np.matmul(grout.reshape(nF, S * F, d), jout).reshape(nF, S, F)
        else:                                      # operator.py:436-444
            uout = 2.0 * self.phys.dirichlet[None, None, :] - uin
            grout, gnout = None, gnin
        dU = uin - uout                                              # (f,q,s)
        gavg_n = 0.5 * (gnin + gnout)                                # (f,s,q)
        sfac = g["sfac"]
        # penalty A_hat . n   (operator.py:336-357)
        if name == "bo":
            q = np.zeros_like(dU)
        elif name == "ip":
            q = (self.eta / g["h"])[:, None, None] * A * dU
        else:
            rin = np.matmul(Pi, dU) * (-0.5 * sfac / self.detJ[ein])[:, None, None]
            if g["interior"]:
                rout = (np.matmul(Po, dU)
                        * (-0.5 * sfac / self.detJ[eout])[:, None, None])
                if name == "br2":
                    rho = 0.5 * (rin + rout)
                else:
                    rho = np.where(g["minus_in"][:, None, None], rin, rout)
            else:
                rho = rin
            fac = 4.0 * self.chi_e if name == "cdg" else 2.0 * self.chi_e
            q = -fac * A * rho
        if self.conv:                                # LLF, flux.py:126-138
            gpin = np.matmul(grin.reshape(nF, S * F, d), self.Jinv[ein])
            gpout = gpin if grout is None else np.matmul(
                grout.reshape(nF, S * F, d), self.Jinv[g["eout"]])
            gav = (0.5 * (gpin + gpout)).reshape(nF, S, F, d).transpose(0, 2, 1, 3)
            lam = self.phys.speed(uin, uout, gav, n[:, None, :])
            Fs = self.phys.flux(uin, gav) + self.phys.flux(uout, gav)   # (f,q,s,d)
            Fn = np.matmul(Fs.reshape(nF, F * S, d), n[:, :, None]).reshape(nF, F, S)
            q = q + 0.5 * Fn + 0.5 * lam[:, :, None] * dU
        wq = (self.wf[None, :] * sfac[:, None])[:, None, :]          # (f,1,q)
        X = wq * dU.transpose(0, 2, 1) * (0.5 * self.adj * A)[None, :, None]
        Y = wq * (gavg_n * A[None, :, None] - q.transpose(0, 2, 1))
        dpin = np.matmul(jin[:, :, 0][:, None, :], self._GfD[g["lin"], g["pin"]]
                         ).reshape(nF, F, -1)                        # (f,q,i)
        out[ein] += np.matmul(Y, Bi) + np.matmul(X, dpin)
        if g["interior"]:
            dpout = np.matmul(jout[:, :, 0][:, None, :],
                              self._GfD[g["lout"], g["pout"]]).reshape(nF, F, -1)
            out[eout] += np.matmul(-Y, Bo) + np.matmul(X, dpout)

    def _wall(self, U, g, out):                    # operator.py:446-458
        B = self.tab[g["lin"], g["pin"]][0]
        ein = g["ein"]
        u = np.einsum("qi,fsi->fqs", B, U[ein])
        q = self.phys.wall(g["tag"], u)
        wq = self.wf[None, :] * g["sfac"][:, None]
        out[ein] -= np.einsum("fq,fqs,qi->fsi", wq, q, B)

    # -- public API (operator.py:253-288) ---------------------------------

    def apply(self, U, t: float = 0.0) -> np.ndarray:
        U = np.asarray(getattr(U, "coeffs", U), dtype=float)
        if U.shape != self.space.shape:
            raise ValueError(f"U has shape {U.shape}, expected "
                             f"{self.space.shape}")
        dirichlet = getattr(self.phys, "dirichlet", None) is not None

        def work(p):
            buf = np.zeros_like(U)
            self._volume(U, self.parts[p], buf)
            for g in self.groups:
                if g["p"] != p:
                    continue
                if g["interior"] or dirichlet:
                    self._faces(U, g, buf)
                else:
                    self._wall(U, g, buf)
            return buf

        if self.nthreads == 1:
            bufs = [work(0)]
        else:
            with ThreadPoolExecutor(self.nthreads) as ex:
                bufs = list(ex.map(work, range(self.nthreads)))
        R = bufs[0]
        for b in bufs[1:]:
            R += b
        return R

    def apply_f(self, U, t: float = 0.0) -> np.ndarray:
        return self.apply(U, t) / self.detJ[:, None, None]


def ssprk3(op, U, dt: float, steps: int):
    """Shu-Osher SSP-RK3 composed from ``apply_f``."""
    U = np.array(U, dtype=float)
    for _ in range(steps):
        U1 = U + dt * op.apply_f(U)
        U2 = 0.75 * U + 0.25 * (U1 + dt * op.apply_f(U1))
        U = U / 3.0 + (2.0 / 3.0) * (U2 + dt * op.apply_f(U2))
    return U


# --------------------------------------------------------- implicit stepper


_SDIRK3_G = 0.435866521508458999416019


def _sdirk3():
    """timeint.py:77-86."""
    g = _SDIRK3_G
    c2 = 0.5 * (1.0 + g)
    b1 = -0.25 * (6.0 * g * g - 16.0 * g + 1.0)
    b2 = 0.25 * (6.0 * g * g - 20.0 * g + 5.0)
    A = np.array([[g, 0.0, 0.0], [c2 - g, g, 0.0], [b1, b2, g]])
    return A, A[-1].copy(), np.array([g, c2, 1.0])


def _gmres(matvec, b, rtol, atol=0.0, restart=30, maxiter=200):
    """Restarted GMRES(m), MGS + Givens (timeint.py:137-207)."""
    n = b.size
    x = np.zeros(n)
    bnorm = float(np.linalg.norm(b))
    target = max(rtol * bnorm, atol)
    if bnorm == 0.0:
        return x, True, 0
    r = b.copy()
    beta = bnorm
    total = 0
    while beta > target and total < maxiter:
        m = min(restart, maxiter - total)
        V = np.empty((m + 1, n))
        H = np.zeros((m + 1, m))
        cs, sn, gv = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        gv[0] = beta
        V[0] = r / beta
        used = 0
        for j in range(m):
            w = matvec(V[j])
            for i in range(j + 1):
                H[i, j] = float(w @ V[i])
                w -= H[i, j] * V[i]
            hn = float(np.linalg.norm(w))
            H[j + 1, j] = hn
            happy = hn <= 1e-14 * max(1.0, float(np.abs(H[:j + 1, j]).max()))
            if not happy:
                V[j + 1] = w / hn
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            rho = math.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if rho == 0.0 else (H[j, j] / rho,
                                                          H[j + 1, j] / rho)
            H[j, j], H[j + 1, j] = rho, 0.0
            gv[j + 1] = -sn[j] * gv[j]
            gv[j] = cs[j] * gv[j]
            used = j + 1
            total += 1
            if abs(gv[j + 1]) <= target or happy:
                break
        y = np.zeros(used)
        for i in range(used - 1, -1, -1):
            y[i] = (gv[i] - H[i, i + 1:used] @ y[i + 1:used]) / H[i, i]
        x = x + y @ V[:used]
        prev = beta
        r = b - matvec(x)
        beta = float(np.linalg.norm(r))
        if beta > 0.99 * prev:
            break
    return x, beta <= target, total


def _newton(G, U0, rtol=1e-8, atol=1e-12, maxiter=25, gmres_rtol=1e-4,
            gmres_restart=30, gmres_maxiter=200):
    """Inexact JFNK Newton (timeint.py:226-289)."""
    U = np.array(U0, dtype=float)
    GU = G(U)
    res = res0 = float(np.linalg.norm(GU))
    target = atol + rtol * res0
    it = 0
    seps = math.sqrt(np.finfo(float).eps)
    while res > target:
        if it >= maxiter:
            raise RuntimeError("Newton did not converge")
        Unorm = float(np.linalg.norm(U))

        def jv(v):
            vn = float(np.linalg.norm(v))
            if vn == 0.0:
                return np.zeros_like(v)
            eps = seps * (1.0 + Unorm) / vn
            return (G(U + eps * v) - GU) / eps

        dU, ok, _ = _gmres(jv, -GU, gmres_rtol, 0.0, gmres_restart,
                           gmres_maxiter)
        if not ok:
            raise RuntimeError("GMRES stalled")
        U = U + dU
        GU = G(U)
        res = float(np.linalg.norm(GU))
        it += 1
    return U


def sdirk_integrate(op, U0, dt: float, n_steps: int, newton_kwargs=None):
    """Fixed-step SDIRK3 (timeint.py:302-380)."""
    A, b, c = _sdirk3()
    U = np.array(U0, dtype=float)
    shape = U.shape
    nk = dict(newton_kwargs or {})
    t = 0.0
    for _ in range(n_steps):
        K = np.empty((3,) + shape)
        for i in range(3):
            base = U + dt * np.einsum("j,j...->...", A[i, :i], K[:i]) \
                if i else U.copy()
            aii = A[i, i]

            def G(v, base=base, aii=aii):
                V = v.reshape(shape)
                return (V - base - dt * aii * op.apply_f(V)).ravel()

            V = _newton(G, base.ravel(), **nk).reshape(shape)
            K[i] = (V - base) / (dt * aii)
        U = U + dt * np.einsum("j,j...->...", b, K)
        t += dt
    return U
