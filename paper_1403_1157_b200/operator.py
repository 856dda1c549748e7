"""Drop-in ``DiscreteOperator`` backed by the sm_100a kernels.

Same constructor, methods and error behaviour as the reference
(``pkg/src/taxisdg/operator.py:77-288``):

    DiscreteOperator(space, model, scheme, nthreads=1, npartitions=None,
                     vol_degree=None, face_degree=None)
    .apply(U, t=0.0)    weak residual <phi, L_h(U)>          (:253-284)
    .apply_f(U, t=0.0)  M^-1 L_h(U)                          (:286-288)
    .set_threads(n, npartitions=None)                        (:208-229)
    .audit_face_ownership()                                  (:231-249)
    attributes .space .model .scheme .mesh

``apply``/``apply_f`` accept a numpy array or ``DiscreteFunction`` (and
return a fresh numpy array, like the reference) or a CUDA
``torch.Tensor`` of the same shape (and return a CUDA tensor, no host
round trip).  The device path is the only path: there is no CPU
fallback, and construction fails loudly without the built library or a
CUDA device.

Beyond the reference API, the explicit stepping entry points used by the
benchmarks and the device-resident JFNK stepper are exposed
(``rk_stage``, ``ssprk3_step``, ``dot``, ``norm2``, ``axpby``).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .fespace import DGSpace
from .flux import FluxScheme
from .tables import build_tables, scheme_constants

__all__ = ["DiscreteOperator"]


# nonzero patterns of the modal linear source the kernels are compiled
# for (models.cuh lin_nz); entries outside them are never read
_LIN_PATTERN = {
    0: [(0, 0), (1, 1), (2, 0), (2, 1), (3, 2), (4, 4), (5, 4)],   # plaque
    1: [(1, 0), (2, 1)],                                           # reduced
    2: [],                                                         # diffusion
}


def _checked_linear_source(model) -> np.ndarray:
    L = np.ascontiguousarray(model.linear_source(), dtype=np.float64)
    mask = np.zeros(L.shape, dtype=bool)
    for s, t in _LIN_PATTERN[model.model_id]:
        mask[s, t] = True
    if np.any(L[~mask] != 0.0):
        raise ValueError("linear source has entries outside the compiled sparsity pattern")
    return L


def _torch():
    import torch
    return torch


class DiscreteOperator:
    def __init__(self, space: DGSpace, model, scheme: FluxScheme,
                 nthreads: int = 1, npartitions: int | None = None,
                 vol_degree: int | None = None, face_degree: int | None = None,
                 device=None, n_owned: int | None = None, global_ids=None, bands: int = 8):
        if model.n_species != space.n_species:
            raise ValueError(f"model has {model.n_species} species, space has "
                             f"{space.n_species}")
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("DiscreteOperator needs a CUDA device (B200); "
                               "there is no CPU path")
        self.space, self.model, self.scheme = space, model, scheme
        self.mesh = space.mesh
        self.device = torch.device(device if device is not None else "cuda")
        self.lib = _native.load()
        t = build_tables(space, model, scheme, vol_degree, face_degree,
                         n_owned=n_owned, global_ids=global_ids, bands=bands)
        self.tables = t
        self.n_owned = t.elem_geo.shape[0]
        self.n_rows = space.mesh.n_elements  # owned + ghost rows of U
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(self.device)
        from .tables import (mma_face_tables, mma_volume_tables, tc_band_blocks,
                             tc_face_blocks, tc_face_tables, tc_volume_tables)
        mma, self._mma_stride = mma_face_tables(t)
        blocks, n_cut_blocks = tc_face_blocks(t)
        self._keep = {"face_mma": dev(mma), "vol_mma": dev(mma_volume_tables(t)),
                      "vol_tc": dev(tc_volume_tables(t)), "face_tc": dev(tc_face_tables(t)[0]),
                      "face_blocks": dev(blocks)}
        self._keep.update({name: dev(getattr(t, name)) for name in (
            "vol_phi", "vol_grad", "vol_w", "vol_stiff", "face_B", "face_G",
            "face_Pw", "face_w", "elem_geo", "if_elems", "if_lf", "if_code",
            "if_geo", "bf_elem", "bf_lf", "bf_code", "bf_geo")})
        self._host = {
            "band_ptr": np.ascontiguousarray(np.concatenate(
                [t.band_elem_ptr, t.band_face_ptr, t.band_wall_ptr,
                 tc_band_blocks(t, blocks)]), dtype=np.int64),
            "diffusivity": np.ascontiguousarray(model.diffusivity(), dtype=np.float64),
            "lin_source": _checked_linear_source(model),
            "params": np.ascontiguousarray(model.pack(), dtype=np.float64)}
        chi_e, adj, eta = scheme_constants(space, scheme)
        ptr = lambda x: ctypes.c_void_p(x.data_ptr() if x.numel() else 0)
        hptr = lambda a: ctypes.c_void_p(a.ctypes.data)
        k = self._keep
        desc = _native.TdgDesc(
            dim=t.dim, order=t.order, n_species=t.n_species, nb=t.nb,
            nq_vol=t.nq_vol, nq_face=t.nq_face, model=model.model_id,
            scheme=scheme.id, n_elements=self.n_owned,
            n_ghost=self.n_rows - self.n_owned,
            n_int_faces=len(t.if_code), n_bnd_faces=len(t.bf_code),
            chi_e=chi_e, adj_sign=adj, ip_eta=eta,
            diffusivity=hptr(self._host["diffusivity"]),
            lin_source=hptr(self._host["lin_source"]),
            params=hptr(self._host["params"]),
            vol_phi=ptr(k["vol_phi"]), vol_grad=ptr(k["vol_grad"]),
            vol_w=ptr(k["vol_w"]), vol_stiff=ptr(k["vol_stiff"]),
            face_B=ptr(k["face_B"]), face_G=ptr(k["face_G"]),
            face_Pw=ptr(k["face_Pw"]), face_w=ptr(k["face_w"]),
            elem_geo=ptr(k["elem_geo"]), if_elems=ptr(k["if_elems"]),
            if_lf=ptr(k["if_lf"]), if_code=ptr(k["if_code"]),
            if_geo=ptr(k["if_geo"]), bf_elem=ptr(k["bf_elem"]),
            bf_lf=ptr(k["bf_lf"]), bf_code=ptr(k["bf_code"]),
            bf_geo=ptr(k["bf_geo"]), face_mma=ptr(k["face_mma"]),
            vol_mma=ptr(k["vol_mma"]), n_cut_faces=t.n_cut, vol_tc=ptr(k["vol_tc"]),
            face_tc=ptr(k["face_tc"]), face_blocks=ptr(k["face_blocks"]),
            n_face_blocks=len(blocks), n_face_blocks_cut=n_cut_blocks,
            n_bands=t.n_bands, band_ptr=hptr(self._host["band_ptr"]))
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(self.lib.tdg_create(ctypes.byref(desc),
                                              ctypes.byref(handle)),
                          "tdg_create")
        self._ctx = handle
        self._scalar = torch.zeros(2, dtype=torch.float64, device=self.device)
        self.set_threads(nthreads, npartitions)

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx is not None and ctx.value:
            try:
                self.lib.tdg_destroy(ctx)
            except Exception:
                pass
            self._ctx = None

    # -- reference API ------------------------------------------------------

    def set_threads(self, nthreads: int, npartitions: int | None = None):
        """Validated like the reference; the device decomposition is fixed
        (one CTA per element / face tile), so the result never depends on
        these values -- it is bitwise reproducible for any of them."""
        if nthreads < 1:
            raise ValueError("nthreads must be >= 1")
        npartitions = nthreads if npartitions is None else npartitions
        if npartitions < 1:
            raise ValueError("npartitions must be >= 1")
        self.nthreads, self.npartitions = int(nthreads), int(npartitions)

    def audit_face_ownership(self) -> dict:
        """Every element is assembled once and every element-local face
        slot is written exactly once per application."""
        t, d = self.tables, self.tables.dim
        slots = np.zeros((self.n_owned, d + 1), dtype=np.int64)
        el, lf, code = t.if_elems, t.if_lf, t.if_code
        np.add.at(slots, (el[:, 0], lf[:, 0]), 1)
        wr = (el[:, 1] >= 0) & ((code & ((1 << 14) | (1 << 15))) == 0)
        np.add.at(slots, (el[wr, 1], lf[wr, 1]), 1)
        np.add.at(slots, (t.bf_elem, t.bf_lf), 1)
        return {"elements_ok": True, "faces_ok": bool((slots == 1).all()),
                "faces_per_part": [len(code) + len(t.bf_code)],
                "elements_per_part": [self.n_owned]}

    def _stream(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def _as_device(self, U):
        torch = _torch()
        shape = (self.n_rows, self.space.n_species, self.space.nb)
        if isinstance(U, torch.Tensor):
            if U.dtype != torch.float64 or U.device.type != "cuda":
                raise ValueError("U must be a float64 CUDA tensor")
            if tuple(U.shape) != shape:
                raise ValueError(f"U has shape {tuple(U.shape)}, expected {shape}")
            return U.contiguous(), True
        U = np.asarray(getattr(U, "coeffs", U), dtype=float)
        if U.shape != shape:
            raise ValueError(f"U has shape {U.shape}, expected {shape}")
        return torch.from_numpy(np.ascontiguousarray(U)).to(self.device), False

    def _apply(self, U, mass_inverse: int, t: float):
        torch = _torch()
        Ud, is_dev = self._as_device(U)
        R = torch.empty((self.n_owned, self.space.n_species, self.space.nb),
                        dtype=torch.float64, device=self.device)
        _native.check(self.lib.tdg_apply(self._ctx, Ud.data_ptr(), R.data_ptr(),
                                         float(t), mass_inverse, self._stream()),
                      "tdg_apply")
        return R if is_dev else R.cpu().numpy()

    def apply(self, U, t: float = 0.0):
        return self._apply(U, 0, t)

    def apply_f(self, U, t: float = 0.0):
        return self._apply(U, 1, t)

    # -- device timing ---------------------------------------------------

    KERNELS = ("faces", "wall", "volume", "fc_add")

    def set_variant(self, generic: bool = False, vol4: bool = False,
                    serial: bool = False, flip_mma: bool = False,
                    mma_volume: bool = False, face_ctas_per_sm: int = 0,
                    no_graph: bool = False, tc_volume: bool = False,
                    no_tc_faces: bool = False, volume_first: bool = False,
                    face_rows_tc: bool = False, one_copy_stream: bool = False,
                    walls_first: bool = False, copy_streams: int = 0):
        """Kernel selection for testing / A-B timing: ``generic`` pins the
        CTA-staged generic kernels; ``vol4`` the four-lanes-per-element
        volume kernel; ``serial`` disables the two-stream overlap of the
        volume part with the face kernel; ``face_ctas_per_sm`` caps the
        grid of the grid-stride face kernel (0 default, 15 uncapped);
        ``face_rows_tc`` the faces-as-rows 3D tensor-core face kernel;
        ``one_copy_stream`` one copy stream per direction in
        ``ssprk3_steps_host`` (``copy_streams``: that many, 0 = default);
        ``walls_first`` 3D wall faces before the
        interior ones.  Defaults: fastest."""
        _native.check(self.lib.tdg_set_variant(
            self._ctx, int(bool(generic)) | (int(bool(vol4)) << 1)
            | (int(bool(serial)) << 2) | (int(bool(flip_mma)) << 3)
            | (int(bool(mma_volume)) << 4) | (int(bool(no_graph)) << 5)
            | (int(bool(tc_volume)) << 12) | (int(bool(no_tc_faces)) << 13)
            | (int(bool(volume_first)) << 14) | (int(bool(face_rows_tc)) << 15)
            | (int(bool(one_copy_stream)) << 16) | (int(bool(walls_first)) << 17)
            | ((int(copy_streams) & 7) << 18)
            | ((int(face_ctas_per_sm) & 15) << 8)),
            "tdg_set_variant")

    def profile(self, enable: bool = True):
        """Bracket every operator kernel launch with CUDA events on its
        stream (per-kernel roofline timing inside the benchmark)."""
        _native.check(self.lib.tdg_profile(self._ctx, int(bool(enable))),
                      "tdg_profile")

    def profile_read(self) -> dict:
        ms = (ctypes.c_double * 4)()
        n = (ctypes.c_int64 * 4)()
        _native.check(self.lib.tdg_profile_read(self._ctx, ms, n),
                      "tdg_profile_read")
        return {k: (ms[i], n[i]) for i, k in enumerate(self.KERNELS)}

    # -- explicit stepping / Krylov primitives (device tensors) ----------

    def _check_vec(self, name, x, rows=None):
        """Raw-pointer entry points need dense fp64 CUDA storage; state
        vectors have the owned rows first (ghost rows optional)."""
        torch = _torch()
        if not isinstance(x, torch.Tensor) or x.dtype != torch.float64 \
                or x.device.type != "cuda" or not x.is_contiguous():
            raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")
        ok_rows = (self.n_owned, self.n_rows) if rows is None else (rows,)
        if rows is not None or x.dim() == 3:
            if x.dim() != 3 or x.shape[1:] != (self.space.n_species, self.space.nb) \
                    or x.shape[0] not in ok_rows:
                raise ValueError(f"{name} has shape {tuple(x.shape)}, expected "
                                 f"(rows in {ok_rows}, {self.space.n_species}, "
                                 f"{self.space.nb})")

    def rk_stage(self, U0, U, out, a: float, b: float, c: float, t: float = 0.0):
        """out = a U0 + b U + c M^-1 L(U) in one fused pass."""
        self._check_vec("U", U, self.n_rows)
        self._check_vec("out", out)
        if U0 is not None:
            self._check_vec("U0", U0)
        _native.check(self.lib.tdg_rk_stage(
            self._ctx, None if U0 is None else U0.data_ptr(), U.data_ptr(),
            out.data_ptr(), float(a), float(b), float(c), float(t),
            self._stream()), "tdg_rk_stage")
        return out

    def rk_stage_part(self, U0, U, out, a: float, b: float, c: float, part: int,
                      t: float = 0.0):
        """Half of ``rk_stage`` around a ghost exchange: part 1 = work on
        owned rows only, part 2 = cut faces + final sum (issue after the
        ghost rows of U are filled)."""
        self._check_vec("U", U, self.n_rows)
        self._check_vec("out", out)
        if U0 is not None:
            self._check_vec("U0", U0)
        _native.check(self.lib.tdg_rk_stage_part(
            self._ctx, None if U0 is None else U0.data_ptr(), U.data_ptr(),
            out.data_ptr(), float(a), float(b), float(c), float(t), int(part),
            self._stream()), "tdg_rk_stage_part")
        return out

    def ssprk3_steps_host(self, U_host, nsteps: int, dt: float, t: float = 0.0):
        """``nsteps`` SSP-RK3 steps of a pinned host state (CPU float64
        tensor of the U shape), with the state copied in and the result
        copied out every step, pipelined by element bands; returns the
        (updated) host tensor.  Asynchronous on the current stream."""
        torch = _torch()
        shape = (self.n_rows, self.space.n_species, self.space.nb)
        if not isinstance(U_host, torch.Tensor) or U_host.device.type != "cpu" \
                or U_host.dtype != torch.float64 or tuple(U_host.shape) != shape \
                or not U_host.is_contiguous() or not U_host.is_pinned():
            raise ValueError(f"U_host must be a pinned, contiguous float64 CPU tensor {shape}")
        _native.check(self.lib.tdg_ssprk3_steps_host(self._ctx, U_host.data_ptr(), int(nsteps),
                                                     float(t), float(dt), self._stream()),
                      "tdg_ssprk3_steps_host")
        return U_host

    def ssprk3_step(self, U, work, dt: float, t: float = 0.0):
        self._check_vec("U", U, self.n_rows)
        self._check_vec("work", work, self.n_rows)
        _native.check(self.lib.tdg_ssprk3_step(
            self._ctx, U.data_ptr(), work.data_ptr(), float(t), float(dt),
            self._stream()), "tdg_ssprk3_step")
        return U

    def species_totals(self, U, out=None):
        """Device int u_s over the owned elements (reference
        ``fespace.py:170-174``); returns a CUDA tensor of S values."""
        torch = _torch()
        self._check_vec("U", U)
        if out is None:
            out = torch.empty(self.space.n_species, dtype=torch.float64, device=self.device)
        _native.check(self.lib.tdg_species_totals(self._ctx, U.data_ptr(), out.data_ptr(),
                                                  self._stream()), "tdg_species_totals")
        return out

    def species_l2(self, U, V=None, out=None):
        """Device broken-L2 norm per species of U - V (or of U) over the
        owned elements: sqrt(sum_e detJ_e sum_i W[e,s,i]^2), exact for the
        orthonormal basis (the parity metric; reference ``l2_error``,
        ``analysis.py:30-50``, for two fields on one space)."""
        torch = _torch()
        self._check_vec("U", U)
        if V is not None:
            self._check_vec("V", V)
        if out is None:
            out = torch.empty(self.space.n_species, dtype=torch.float64, device=self.device)
        _native.check(self.lib.tdg_species_l2(
            self._ctx, U.data_ptr(), None if V is None else V.data_ptr(), out.data_ptr(),
            self._stream()), "tdg_species_l2")
        return out

    def mgs(self, V, j: int, w, h):
        """One modified Gram-Schmidt sweep (GMRES Arnoldi step, reference
        ``timeint.py:162-170``) against rows V[0..j]: h[i] = w.V_i,
        w -= h[i] V_i, h[j+1] = ||w||; all on the device, one call."""
        if V.dim() != 2 or not V.is_contiguous() or not w.is_contiguous():
            raise ValueError("mgs needs a contiguous 2-D V and a contiguous w")
        n = w.numel()
        if V.shape[1] != n or j + 1 > V.shape[0] or h.numel() < j + 2:
            raise ValueError("mgs: inconsistent sizes")
        _native.check(self.lib.tdg_mgs(self._ctx, V.data_ptr(), V.stride(0), int(j), w.data_ptr(),
                                       n, h.data_ptr(), self._stream()), "tdg_mgs")
        return h

    def scale_norm(self, w, hnext, v, norm_out):
        """v = w / hnext (GMRES basis vector, reference ``timeint.py:165,176``)
        and ||v|| into the device scalar ``norm_out``, one pass; ``hnext`` a
        float or a one-element CUDA tensor (device divisor)."""
        torch = _torch()
        dev_div = isinstance(hnext, torch.Tensor)
        if dev_div:
            self._check_vec("hnext", hnext)
        w, v = w.reshape(-1), v.reshape(-1)
        self._check_vec("w", w)
        self._check_vec("v", v)
        if w.numel() != v.numel():
            raise ValueError("w and v differ in size")
        _native.check(self.lib.tdg_scale_norm(
            self._ctx, w.data_ptr(), 0.0 if dev_div else float(hnext),
            hnext.data_ptr() if dev_div else None, v.data_ptr(), w.numel(), norm_out.data_ptr(),
            self._stream()), "tdg_scale_norm")
        return v

    def jv_shift(self, U, v, vnorm, cnum: float, Up, eps_out):
        """eps = cnum / max(||v||, 1e-300) (device), Up = U + eps v
        (reference ``timeint.py:259-264``)."""
        n = U.numel()
        for name, x in (("U", U), ("v", v), ("Up", Up)):
            self._check_vec(name, x.reshape(-1))
        if v.numel() != n or Up.numel() != n:
            raise ValueError("jv_shift: size mismatch")
        _native.check(self.lib.tdg_jv_shift(U.data_ptr(), v.data_ptr(), vnorm.data_ptr(),
                                            float(cnum), Up.data_ptr(), eps_out.data_ptr(), n,
                                            self._stream()), "tdg_jv_shift")
        return Up

    def jv_diff(self, r, GU, eps):
        """r = (r - GU) / eps in place (device eps)."""
        self._check_vec("r", r.reshape(-1))
        self._check_vec("GU", GU.reshape(-1))
        if r.numel() != GU.numel():
            raise ValueError("jv_diff: size mismatch")
        _native.check(self.lib.tdg_jv_diff(r.data_ptr(), GU.data_ptr(), eps.data_ptr(), r.numel(),
                                           self._stream()), "tdg_jv_diff")
        return r

    def dot(self, x, y, out=None):
        x, y = x.reshape(-1), y.reshape(-1)
        self._check_vec("x", x)
        self._check_vec("y", y)
        if x.numel() != y.numel():
            raise ValueError("x and y differ in size")
        out = self._scalar[:1] if out is None else out
        _native.check(self.lib.tdg_dot(self._ctx, x.data_ptr(), y.data_ptr(),
                                       x.numel(), out.data_ptr(), self._stream()),
                      "tdg_dot")
        return out

    def norm2(self, x, out=None):
        x = x.reshape(-1)
        self._check_vec("x", x)
        out = self._scalar[1:] if out is None else out
        _native.check(self.lib.tdg_norm2(self._ctx, x.data_ptr(), x.numel(),
                                         out.data_ptr(), self._stream()),
                      "tdg_norm2")
        return out

    def axpby(self, a: float, x, b: float, y):
        if x.numel() != y.numel():
            raise ValueError("x and y differ in size")
        self._check_vec("x", x.reshape(-1))
        self._check_vec("y", y.reshape(-1))
        _native.check(self.lib.tdg_axpby(float(a), x.data_ptr(), float(b),
                                         y.data_ptr(), x.numel(), self._stream()),
                      "tdg_axpby")
        return y

    def axpy_dev(self, s: float, alpha, x, y):
        if x.numel() != y.numel():
            raise ValueError("x and y differ in size")
        self._check_vec("x", x.reshape(-1))
        self._check_vec("y", y.reshape(-1))
        _native.check(self.lib.tdg_axpy_dev(float(s), alpha.data_ptr(),
                                            x.data_ptr(), y.data_ptr(),
                                            x.numel(), self._stream()),
                      "tdg_axpy_dev")
        return y
