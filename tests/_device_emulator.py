"""numpy emulation of the CUDA kernels' arithmetic (test infrastructure).

Consumes the same packed ``OperatorTables`` the device gets and performs
the kernels' reformulated operation sequence (csrc/kernels.cuh,
csrc/models.cuh).  Lets the CPU suite check the reformulation against the
oracle without a GPU; the GPU suite then checks the kernels against both.
"""
import numpy as np

from paper_1403_1157_b200.model import MODEL_DIFFUSION, MODEL_PLAQUE, \
    MODEL_REDUCED
from paper_1403_1157_b200.tables import sym_pairs

CIN, MIRROR, SKIP, FIRST_IN, FIRST_OUT = 1 << 10, 1 << 14, 1 << 15, 1 << 16, 1 << 17


def _plaque_volume(P, v, gM):
    n1, n2, c1, c3 = v
    x11 = P[13] * n1 / (np.maximum(c1, 0) + P[14])
    x13 = P[15] * n1 / (np.maximum(c3, 0) + P[16])
    x21 = P[17] * n2 / (np.maximum(c1, 0) + P[18])
    x2n = P[19] * n2 / (np.maximum(n1, 0) + P[20])
    f0 = x11[:, None] * gM[1] + x13[:, None] * gM[2]
    f1 = x21[:, None] * gM[1] - x2n[:, None] * gM[0]
    nl = -P[8] * n1 * c1 - P[9] * n2 * c1
    return [f0, f1], [nl]


def _heav(s, eps):
    if eps == 0.0:
        return (s > 0).astype(float)
    return 1.0 / (1.0 + np.exp(np.clip(-s / eps, -60, 60)))


class DeviceEmulator:
    def __init__(self, tables, model, scheme, chi_e, adj, eta, normal_after=False):
        # normal_after: the signature-run kernel's order (k_faces_sig): the
        # normal derivative after the contraction, jn . (G c), and the adjoint
        # term projected with (X jn) . G instead of a per-face d_n phi table
        self.normal_after = normal_after
        self.t, self.model, self.scheme = tables, model, scheme
        self.chi_e, self.adj, self.eta = chi_e, adj, eta
        self.A = model.diffusivity()
        self.L = model.linear_source()
        self.P = model.pack()
        self.mid = model.model_id

    def apply(self, U):
        """Face segments in order (each face side writes or adds to its
        element's face-sum row per its FIRST flag; no element twice in a
        segment), then the volume terms plus the face sums."""
        t = self.t
        S, nb = t.n_species, t.nb
        ne = t.elem_geo.shape[0]
        ACC = np.full((ne, S, nb), np.nan)
        for s in range(t.n_seg):
            seen = set()

            def put(e, v, first):
                assert e not in seen, f"element {e} written twice in segment {s}"
                seen.add(e)
                if first:
                    ACC[e] = v
                else:
                    assert np.isfinite(ACC[e]).all(), f"element {e}: add before first write"
                    ACC[e] += v

            for f in range(t.seg_if[s], t.seg_if[s + 1]):
                code = int(t.if_code[f])
                ein, eout = t.if_elems[f]
                ri, ro = self.face_contrib(U, code, ein, eout, t.if_geo[f])
                put(ein, ri, bool(code & FIRST_IN))
                if ro is not None and not (code & SKIP):
                    put(eout, ro, bool(code & FIRST_OUT))
            for f in range(t.seg_bf[s], t.seg_bf[s + 1]):
                code = int(t.bf_code[f])
                put(t.bf_elem[f], self.wall_contrib(U, code, t.bf_elem[f], t.bf_geo[f]),
                    bool(code & FIRST_IN))
        return self._volume(U, ACC)

    def _volume(self, U, FC):
        t = self.t
        d, nb = t.dim, t.nb
        ne = t.elem_geo.shape[0]
        c = U[:ne]
        detJ = t.elem_geo[:, 0]
        Msym = t.elem_geo[:, 1:]
        Kp = np.einsum("ep,pji->eji", Msym, t.vol_stiff)
        R = -self.A[None, :, None] * np.einsum("esj,eji->esi", c, Kp)
        R += np.einsum("st,eti->esi", self.L, c)
        if self.mid in (MODEL_PLAQUE, MODEL_REDUCED):
            phi, gr, w = t.vol_phi, t.vol_grad, t.vol_w
            Mfull = np.zeros((ne, d, d))
            for p, (a, b) in enumerate(sym_pairs(d)):
                Mfull[:, a, b] = Msym[:, p]
                Mfull[:, b, a] = Msym[:, p]
            for q in range(len(w)):
                if self.mid == MODEL_PLAQUE:
                    v = [c[:, s] @ phi[q] for s in (0, 1, 3, 5)]
                    g = [np.einsum("ei,ia->ea", c[:, s], gr[q]) for s in (0, 3, 5)]
                    gM = [np.einsum("ea,eab->eb", x, Mfull) for x in g]
                    fr, nl = _plaque_volume(self.P, v, gM)
                    fsp, nsp = (0, 1), 3
                else:
                    P = self.P
                    n1, c1 = c[:, 0] @ phi[q], c[:, 2] @ phi[q]
                    gc1 = np.einsum("ei,ia->ea", c[:, 2], gr[q])
                    gM = np.einsum("ea,eab->eb", gc1, Mfull)
                    fr = [(P[13] * n1 / (np.maximum(c1, 0) + P[14]))[:, None] * gM]
                    nl = [-P[8] * n1 * c1]
                    fsp, nsp = (0,), 2
                for k, s in enumerate(fsp):
                    R[:, s] += w[q] * np.einsum("ea,ia->ei", fr[k], gr[q])
                R[:, nsp] += w[q] * nl[0][:, None] * phi[q][None, :]
        R = detJ[:, None, None] * R
        if FC is not None:
            R = R + FC
        return R

    def _conv(self, ui, uo, gn, dU, qv):
        P = self.P
        if self.mid == MODEL_PLAQUE:
            lam = np.zeros(ui.shape[0])
            f0 = np.zeros_like(lam)
            f1 = np.zeros_like(lam)
            for u in (ui, uo):
                c1p = np.maximum(u[:, 3], 0)
                v0 = P[13] / (c1p + P[14]) * gn[:, 3] + P[15] / (np.maximum(u[:, 5], 0) + P[16]) * gn[:, 5]
                v1 = P[17] / (c1p + P[18]) * gn[:, 3] - P[19] / (np.maximum(u[:, 0], 0) + P[20]) * gn[:, 0]
                lam = np.maximum(lam, np.maximum(abs(v0), abs(v1)))
                f0 += u[:, 0] * v0
                f1 += u[:, 1] * v1
            qv[:, 0] += 0.5 * f0
            qv[:, 1] += 0.5 * f1
            qv += 0.5 * lam[:, None] * dU
        elif self.mid == MODEL_REDUCED:
            lam = np.zeros(ui.shape[0])
            f0 = np.zeros_like(lam)
            for u in (ui, uo):
                v0 = P[13] / (np.maximum(u[:, 2], 0) + P[14]) * gn[:, 2]
                lam = np.maximum(lam, abs(v0))
                f0 += u[:, 0] * v0
            qv[:, 0] += 0.5 * f0
            qv += 0.5 * lam[:, None] * dU

    def face_contrib(self, U, code, ein, eout, g):
        """(inside row, outside row or None) of one interior/mirror face."""
        t = self.t
        d, S, nb = t.dim, t.n_species, t.nb
        F = t.nq_face
        if True:
            tin, tout = code & 31, (code >> 5) & 31
            mirror = bool(code & MIRROR)
            jin, jout = g[:d], g[d:2 * d]
            sfac, h, idi, ido = g[2 * d:2 * d + 4]
            dpi = np.einsum("qia,a->qi", t.face_G[tin], jin)
            ci = U[ein]
            ui = ci @ t.face_B[tin].T          # (S, F)
            gi = ci @ dpi.T
            after = self.normal_after and not mirror
            if after:
                gi = np.einsum("sqa,a->sq", np.einsum("si,qia->sqa", ci, t.face_G[tin]), jin)
            if mirror:
                gval = self.P[:S]
                uo = 2 * gval[:, None] - ui
                go = gi
            else:
                dpo = np.einsum("qia,a->qi", t.face_G[tout], jout)
                co = U[eout]
                uo = co @ t.face_B[tout].T
                go = co @ dpo.T
                if after:
                    go = np.einsum("sqa,a->sq",
                                   np.einsum("si,qia->sqa", co, t.face_G[tout]), jout)
            dU = ui - uo
            gn = 0.5 * (gi + go)
            qv = np.zeros((F, S))
            name = self.scheme
            if name == 3:
                qv = (self.eta / h) * self.A[None, :] * dU.T
            elif name != 4:
                br2 = name == 2
                use_in = mirror or br2 or bool(code & CIN)
                use_out = (not mirror) and (br2 or not (code & CIN))
                wside = 0.5 if (br2 and not mirror) else 1.0
                rho = np.zeros((S, F))
                if use_in:
                    rho += wside * (-0.5 * sfac * idi) * (dU @ t.face_Pw[tin].T)
                if use_out:
                    rho += wside * (-0.5 * sfac * ido) * (dU @ t.face_Pw[tout].T)
                fac = (4.0 if name == 1 else 2.0) * self.chi_e
                qv = (-fac * self.A[:, None] * rho).T
            self._conv(ui.T, uo.T, gn.T, dU.T, qv)
            wq = t.face_w * sfac
            Y = wq[None, :] * (self.A[:, None] * gn - qv.T)
            X = wq[None, :] * 0.5 * self.adj * self.A[:, None] * dU
            if after:
                ri = Y @ t.face_B[tin] + np.einsum("sqa,qia->si", X[:, :, None] * jin,
                                                   t.face_G[tin])
                ro = -Y @ t.face_B[tout] + np.einsum("sqa,qia->si", X[:, :, None] * jout,
                                                     t.face_G[tout])
                return ri, ro
            ri = Y @ t.face_B[tin] + X @ dpi
            ro = None if mirror else -Y @ t.face_B[tout] + X @ dpo
            return ri, ro

    def wall_contrib(self, U, code, e, sfac):
        t = self.t
        S = t.n_species
        P = self.P
        if True:
            tin, tag = code & 31, (code >> 11) & 7
            B = t.face_B[tin]
            q = np.zeros((S, t.nq_face))
            if self.mid == MODEL_PLAQUE:
                c1 = B @ U[e, 3]
                if tag in (1, 2):
                    q[0] = -P[0] * P[21] * _heav(c1 - P[24], P[26])
                if tag == 2:
                    q[4] = -P[4] * P[23]
                if tag == 3:
                    q[1] = -P[1] * P[22] * _heav(c1 - P[25], P[26])
            elif self.mid == MODEL_REDUCED:
                c1 = B @ U[e, 2]
                if tag in (1, 2):
                    q[0] = -P[0] * P[21] * _heav(c1 - P[24], P[26])
            Y = -(t.face_w * sfac)[None, :] * q
            return Y @ B
