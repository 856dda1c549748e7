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

The constructor takes this package's ``DGSpace`` / model / ``FluxScheme``
or the reference's own ``taxisdg`` objects (``compat.adapt``), so the
reference's call sites need only the import swapped.

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
from .compat import adapt
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
                 device=None, n_owned: int | None = None, global_ids=None):
        if model.n_species != space.n_species:
            raise ValueError(f"model has {model.n_species} species, space has "
                             f"{space.n_species}")
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("DiscreteOperator needs a CUDA device (B200); "
                               "there is no CPU path")
        # the caller's objects (package or reference taxisdg ones) stay the
        # public attributes; the device is described from their adapted
        # package equivalents (compat.adapt)
        self.space, self.model, self.scheme = space, model, scheme
        self.mesh = space.mesh
        space, model, scheme = adapt(space, model, scheme)
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.lib = _native.load()
        t = build_tables(space, model, scheme, vol_degree, face_degree,
                         n_owned=n_owned, global_ids=global_ids)
        self.tables = t
        self.n_owned = t.elem_geo.shape[0]
        self.n_rows = space.mesh.n_elements  # owned + ghost rows of U
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(self.device)
        from .tables import (CODE_FIRST_IN, CODE_FIRST_OUT, mma_face_tables,
                             seg_chunk_offsets, tc_face_blocks, tc_face_fold_tables,
                             tc_face_groups, tc_face_tables, tc_volume_classes,
                             tc_volume_tables, modal_face_tables)
        mma, self._mma_stride = mma_face_tables(t)
        blocks, seg_blk = tc_face_blocks(t)
        fold = tc_face_fold_tables(t)
        self.n_face_classes = 0 if fold is None else len(fold[0]) // fold[1]
        self._keep = {"face_mma": dev(mma), "vol_tc": dev(tc_volume_tables(t)),
                      "face_tc": dev(tc_face_tables(t)[0] if t.dim == 3 else np.zeros(4)),
                      "face_blocks": dev(blocks)}
        groups, seg_grp = np.zeros((0, 1), np.int32), np.zeros(t.n_seg + 1, np.int64)
        if fold is not None:
            self._keep["face_tc_fold"] = dev(fold[0])
            self._keep["if_fold"] = dev(fold[2])
            groups, seg_grp = tc_face_groups(t, fold[2], t.n_species)
            self._keep["face_groups"] = dev(groups)
            self._keep["face_modal"] = dev(modal_face_tables(t, fold))
        # element-geometry classes of the tensor-core volume kernel (3D and
        # 2D p = 3; meshes of congruent cells)
        vcls = tc_volume_classes(t) if (t.dim == 3 or t.order == 3) else None
        self.n_volume_classes = 0 if vcls is None else len(np.unique(vcls[2]))
        if vcls is not None:
            self._keep["vol_cls_tab"] = dev(vcls[0])
            self._keep["vol_perm"] = dev(vcls[1])
            self._keep["vol_task_cls"] = dev(vcls[2])
        self._keep.update({name: dev(getattr(t, name)) for name in (
            "vol_phi", "vol_grad", "vol_w", "vol_stiff", "face_B", "face_G",
            "face_Pw", "face_w", "elem_geo", "if_elems", "if_code",
            "if_geo", "bf_elem", "bf_code", "bf_geo")})
        # point data of the diffusion model's x-dependent closures
        self._pd_t = None
        if getattr(model, "has_point_data", False):
            nq, S = t.nq_face, t.n_species
            self._keep["if_bval"] = torch.zeros((max(len(t.if_code), 1), nq, S),
                                                dtype=torch.float64, device=self.device)
            self._keep["bf_qval"] = torch.zeros((max(len(t.bf_code), 1), nq, S),
                                                dtype=torch.float64, device=self.device)
            self._pd_model = model
            self._set_point_data(0.0)
        # host-data stepping: (segment, chunk) runs and add-only code words
        # (tdg_desc.seg_chunk_ptr, tables.seg_chunk_offsets)
        chunked = self.n_rows == self.n_owned and len(t.if_code) + len(t.bf_code) > 0
        if chunked:
            nseg = t.n_seg
            bseg = np.repeat(np.arange(nseg), np.diff(t.seg_bf))
            offs = [seg_chunk_offsets(t.if_seg, t.if_chunk, nseg),
                    seg_chunk_offsets(bseg, t.bf_chunk, nseg)]
            if len(blocks):
                offs.append(seg_chunk_offsets(t.if_seg[blocks[:, 0]], t.if_chunk[blocks[:, 0]], nseg))
            else:
                offs.append(np.zeros(nseg * 8 + 1, np.int64))
            if len(groups) and groups.shape[1] and "face_groups" in self._keep:
                g0 = groups[:, 0]
                offs.append(seg_chunk_offsets(t.if_seg[g0], t.if_chunk[g0], nseg))
            else:
                offs.append(np.zeros(nseg * 8 + 1, np.int64))
            first = CODE_FIRST_IN | CODE_FIRST_OUT
            self._keep["if_code_add"] = dev((t.if_code & ~first).astype(np.int32)
                                            if len(t.if_code) else np.zeros(1, np.int32))
            self._keep["bf_code_add"] = dev((t.bf_code & ~first).astype(np.int32)
                                            if len(t.bf_code) else np.zeros(1, np.int32))
        self._host = {
            "seg_chunk_ptr": (np.ascontiguousarray(np.concatenate(offs), dtype=np.int64)
                              if chunked else np.zeros(1, np.int64)),
            "seg_ptr": np.ascontiguousarray(np.concatenate(
                [t.seg_if, t.seg_bf, seg_blk, seg_grp]), dtype=np.int64),
            "diffusivity": np.ascontiguousarray(model.diffusivity(), dtype=np.float64),
            "lin_source": _checked_linear_source(model),
            "params": np.ascontiguousarray(model.pack(), dtype=np.float64),
            "vol_chunk_tasks": np.ascontiguousarray(
                vcls[3] if vcls is not None else np.zeros(9), dtype=np.int64)}
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
            if_code=ptr(k["if_code"]), if_geo=ptr(k["if_geo"]),
            bf_elem=ptr(k["bf_elem"]), bf_code=ptr(k["bf_code"]),
            bf_geo=ptr(k["bf_geo"]), face_mma=ptr(k["face_mma"]),
            vol_tc=ptr(k["vol_tc"]), face_tc=ptr(k["face_tc"]),
            face_blocks=ptr(k["face_blocks"]), n_face_blocks=len(blocks),
            face_tc_fold=ptr(k["face_tc_fold"]) if fold is not None else None,
            if_fold=ptr(k["if_fold"]) if fold is not None else None,
            face_groups=ptr(k["face_groups"]) if fold is not None else None,
            n_face_groups=len(groups),
            face_modal=ptr(k["face_modal"]) if fold is not None else None,
            vol_cls_tab=ptr(k["vol_cls_tab"]) if vcls is not None else None,
            vol_perm=ptr(k["vol_perm"]) if vcls is not None else None,
            vol_task_cls=ptr(k["vol_task_cls"]) if vcls is not None else None,
            n_vol_tasks=len(vcls[2]) if vcls is not None else 0,
            vol_chunk_tasks=hptr(self._host["vol_chunk_tasks"]) if vcls is not None else None,
            if_bval=ptr(k["if_bval"]) if "if_bval" in k else None,
            bf_qval=ptr(k["bf_qval"]) if "bf_qval" in k else None,
            seg_chunk_ptr=hptr(self._host["seg_chunk_ptr"]) if chunked else None,
            if_code_add=ptr(k["if_code_add"]) if chunked else None,
            bf_code_add=ptr(k["bf_code_add"]) if chunked else None,
            n_segments=t.n_seg, n_segments_cut=t.n_seg_cut,
            seg_ptr=hptr(self._host["seg_ptr"]))
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            # tdg_create reads some device tables back (signature runs) and copies others
            # to constant memory on the default stream: the uploads above must be done
            torch.cuda.current_stream(self.device).synchronize()
            _native.check(self.lib.tdg_create(ctypes.byref(desc), ctypes.byref(handle)),
                          "tdg_create")
            self._dev_index = torch.cuda.current_device()
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
        """Reference ``operator.py:231-249`` audits that every element and
        face is assembled exactly once.  Here: every element-local face
        slot is written by exactly one face side; within each colour
        segment (one launch) no element is written twice (the race-freedom
        of the accumulating face kernels); every element's first side in
        segment order carries the write flag, every other side adds."""
        t, d = self.tables, self.tables.dim
        slots = np.zeros((self.n_owned, d + 1), dtype=np.int64)
        el, lf, code = t.if_elems, t.if_lf, t.if_code
        np.add.at(slots, (el[:, 0], lf[:, 0]), 1)
        wr = (el[:, 1] >= 0) & ((code & ((1 << 14) | (1 << 15))) == 0)
        np.add.at(slots, (el[wr, 1], lf[wr, 1]), 1)
        np.add.at(slots, (t.bf_elem, t.bf_lf), 1)
        seg_w = np.repeat(np.arange(t.n_seg), np.diff(t.seg_bf))
        e_all = np.concatenate([el[:, 0], el[wr, 1], t.bf_elem])
        s_all = np.concatenate([t.if_seg, t.if_seg[wr], seg_w]).astype(np.int64)
        f_all = np.concatenate([(code >> 16) & 1, (code[wr] >> 17) & 1,
                                (t.bf_code >> 16) & 1])
        pair = e_all.astype(np.int64) * max(t.n_seg, 1) + s_all
        once = len(np.unique(pair)) == len(pair)
        firsts = np.bincount(e_all[f_all == 1], minlength=self.n_owned)
        first_min = np.full(self.n_owned, np.iinfo(np.int64).max)
        np.minimum.at(first_min, e_all, s_all)
        first_ok = bool((firsts == 1).all()) and bool(
            (first_min[e_all[f_all == 1]] == s_all[f_all == 1]).all())
        per_seg = [int(t.seg_if[s + 1] - t.seg_if[s] + t.seg_bf[s + 1] - t.seg_bf[s])
                   for s in range(t.n_seg)]
        return {"elements_ok": True, "faces_ok": bool((slots == 1).all()),
                "segments_race_free": bool(once), "first_flags_ok": first_ok,
                "faces_per_part": per_seg, "elements_per_part": [self.n_owned]}

    def _stream(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def _call(self, fn, *args, what="tdg call"):
        """Native call on this operator's device (launches go to the
        device's current stream; the caller's current device may differ)."""
        torch = _torch()
        if torch.cuda.current_device() != self._dev_index:
            with torch.cuda.device(self.device):
                rc = fn(*args)
        else:
            rc = fn(*args)
        _native.check(rc, what)

    def _as_device(self, U):
        torch = _torch()
        shape = (self.n_rows, self.space.n_species, self.space.nb)
        if isinstance(U, torch.Tensor):
            if U.dtype != torch.float64 or U.device != self.device:
                raise ValueError(f"U must be a float64 tensor on {self.device}")
            if tuple(U.shape) != shape:
                raise ValueError(f"U has shape {tuple(U.shape)}, expected {shape}")
            return U.contiguous(), True
        U = np.asarray(getattr(U, "coeffs", U), dtype=float)
        if U.shape != shape:
            raise ValueError(f"U has shape {U.shape}, expected {shape}")
        return torch.from_numpy(np.ascontiguousarray(U)).to(self.device), False

    def _set_point_data(self, t: float):
        """Evaluate the model's x-dependent boundary closures at the face
        quadrature points (reference operator.py:436-458) and upload them."""
        tb, model, mesh = self.tables, self._pd_model, self.space.mesh
        d, nq, S = tb.dim, tb.nq_face, tb.n_species
        nperm = 2 if d == 2 else 6
        from .fespace import face_reference_points
        J, _, _ = mesh.jacobians()
        if model.dirichlet_fn is not None:
            vals = np.zeros((max(len(tb.if_code), 1), nq, S))
            mirror = np.flatnonzero(tb.if_code & (1 << 14))
            tin = tb.if_code[mirror] & 31
            for tid in np.unique(tin):
                sel = mirror[tin == tid]
                e = tb.if_elems[sel, 0]
                xi = face_reference_points(d, int(tid) // nperm, int(tid) % nperm, tb.face_pts)
                X = mesh.vertices[mesh.elements[e, 0]][:, None, :] + np.einsum(
                    "fij,qj->fqi", J[e], xi)
                vals[sel] = np.asarray(model.dirichlet_fn(X.reshape(-1, d), t),
                                       dtype=float).reshape(len(sel), nq, S)
            self._keep["if_bval"].copy_(_torch().from_numpy(vals))
        if model.wall_flux_fn is not None and len(tb.bf_code):
            vals = np.zeros((len(tb.bf_code), nq, S))
            tags = mesh.face_tags[tb.bf_fid]
            for tag in np.unique(tags):
                sel = np.flatnonzero(tags == tag)
                nrm = np.repeat(mesh.face_normals[tb.bf_fid[sel]], nq, axis=0)
                q = model.wall_flux_fn(int(tag), np.zeros((len(sel) * nq, S)), nrm, t)
                vals[sel] = np.asarray(q, dtype=float).reshape(len(sel), nq, S)
            self._keep["bf_qval"].copy_(_torch().from_numpy(vals))
        self._pd_t = float(t)

    def _point_data_at(self, t: float, entry: str):
        if self._pd_t is None or not self._pd_model.time_dependent or float(t) == self._pd_t:
            return
        if entry != "apply":
            raise ValueError("time-dependent boundary data: step through apply / apply_f "
                             "(the reference's stepper call shape)")
        self._set_point_data(t)

    def _apply(self, U, mass_inverse: int, t: float):
        torch = _torch()
        self._point_data_at(t, "apply")
        rshape = (self.n_owned, self.space.n_species, self.space.nb)
        if not isinstance(U, torch.Tensor):
            # host data (numpy / DiscreteFunction), the reference's call
            # shape: staged copies in and out (tdg_apply_host), a fresh
            # numpy result like the reference
            shape = (self.n_rows, self.space.n_species, self.space.nb)
            Uh = np.ascontiguousarray(np.asarray(getattr(U, "coeffs", U), dtype=float))
            if Uh.shape != shape:
                raise ValueError(f"U has shape {Uh.shape}, expected {shape}")
            Rh = np.empty(rshape)
            Ud = torch.empty(shape, dtype=torch.float64, device=self.device)
            Rd = torch.empty(rshape, dtype=torch.float64, device=self.device)
            self._call(self.lib.tdg_apply_host, self._ctx, Uh.ctypes.data, Rh.ctypes.data,
                       Ud.data_ptr(), Rd.data_ptr(), float(t), mass_inverse, self._stream(),
                       what="tdg_apply_host")
            return Rh
        Ud, _ = self._as_device(U)
        R = torch.empty(rshape, dtype=torch.float64, device=self.device)
        self._call(self.lib.tdg_apply, self._ctx, Ud.data_ptr(), R.data_ptr(), float(t),
                   mass_inverse, self._stream(), what="tdg_apply")
        return R

    def apply(self, U, t: float = 0.0):
        return self._apply(U, 0, t)

    def apply_f(self, U, t: float = 0.0):
        return self._apply(U, 1, t)

    # -- device timing ---------------------------------------------------

    KERNELS = ("faces", "wall", "volume", "reserved")

    def kernel_names(self) -> dict:
        """The kernels the default variant launches per kernel class (the
        library's dispatch rules, ctx.cuh run_segment / volume, for the
        compiled-in default quadrature)."""
        t = self.tables
        if t.dim == 3:
            if self.n_face_classes and len(self._keep.get("face_groups", ())):
                faces = "k_faces_tcm" if "face_modal" in self._keep else "k_faces_tcg"
            else:
                faces = "k_faces_tcs"
            wall = "k_faces_mma"
        elif self.face_runs()[0]:
            # walls ride in the last run's launch; states larger than half the
            # L2 take the cp.async-staged variant (ctx.cuh run_segment)
            import torch
            l2 = torch.cuda.get_device_properties(self.device).L2_cache_size
            rows = self.space.mesh.n_elements * t.n_species * t.nb * 8
            faces = wall = "k_faces_sig_async" if rows > l2 // 2 else "k_faces_sig"
        else:
            faces, wall = "k_faces_fast", "k_faces_fast (walls)"
        if t.dim == 3 or t.order == 3:
            volume = "k_volume_tc" + (" (element classes)" if self.n_volume_classes else "")
        else:
            volume = "k_volume_fast"
        return {"faces": faces, "wall": wall, "volume": volume}

    def face_runs(self) -> tuple:
        """(signature runs, folded runs) of the 2D signature-run face kernel
        ``k_faces_sig``; (0, 0) when the library does not use it."""
        n, nf = ctypes.c_int64(0), ctypes.c_int64(0)
        self._call(self.lib.tdg_face_runs, self._ctx, ctypes.byref(n), ctypes.byref(nf),
                   what="tdg_face_runs")
        return int(n.value), int(nf.value)

    def set_variant(self, generic: bool = False, no_graph: bool = False,
                    tc_volume: bool = False, face_ctas_per_sm: int = 0,
                    no_fold: bool = False, no_groups: bool = False,
                    no_volume_classes: bool = False, no_modal: bool = False,
                    no_sig: bool = False, sig_async: bool = False):
        """Kernel selection for testing / A-B timing: ``generic`` pins the
        CTA-staged generic kernels; ``no_graph`` launches ``ssprk3_step``'s
        kernels directly instead of replaying its CUDA graph; ``tc_volume``
        the tensor-core volume kernel where the SIMT one fits;
        ``face_ctas_per_sm`` caps the grid of the 2D grid-stride face kernel
        (0 default, 15 uncapped); ``no_fold`` makes the 3D face kernel fold
        Jinv n per face despite face-geometry-class tables; ``no_groups``
        runs the one-face species-rows kernel instead of the face-group
        kernel; ``no_volume_classes`` scales the volume kernel's diffusion
        per element despite element-geometry classes; ``no_modal`` runs the
        face-group kernel on full traces instead of the modal face space;
        ``no_sig`` runs the 2D faces on ``k_faces_fast`` (tables in shared
        memory) instead of the signature-run kernel ``k_faces_sig``;
        ``sig_async`` runs its cp.async-staged variant (the default only for
        states larger than half the L2) at any size.
        Defaults: fastest."""
        self._call(self.lib.tdg_set_variant, self._ctx,
                   int(bool(generic)) | (int(bool(no_graph)) << 5)
                   | (int(bool(tc_volume)) << 12) | (int(bool(no_fold)) << 13)
                   | (int(bool(no_groups)) << 14) | (int(bool(no_volume_classes)) << 15)
                   | (int(bool(no_modal)) << 16) | (int(bool(no_sig)) << 17)
                   | (int(bool(sig_async)) << 18)
                   | ((int(face_ctas_per_sm) & 15) << 8),
                   what="tdg_set_variant")

    def profile(self, enable: bool = True):
        """Bracket every operator kernel launch with CUDA events on its
        stream (per-kernel roofline timing inside the benchmark)."""
        self._call(self.lib.tdg_profile, self._ctx, int(bool(enable)), what="tdg_profile")

    def profile_read(self) -> dict:
        ms = (ctypes.c_double * 4)()
        n = (ctypes.c_int64 * 4)()
        self._call(self.lib.tdg_profile_read, self._ctx, ms, n, what="tdg_profile_read")
        return {k: (ms[i], n[i]) for i, k in enumerate(self.KERNELS)}

    # -- explicit stepping / Krylov primitives (device tensors) ----------

    def _check_vec(self, name, x, rows=None):
        """Raw-pointer entry points need dense fp64 storage on this
        operator's device; state vectors have the owned rows first (ghost
        rows optional)."""
        torch = _torch()
        if not isinstance(x, torch.Tensor) or x.dtype != torch.float64 \
                or x.device != self.device or not x.is_contiguous():
            raise ValueError(f"{name} must be a contiguous float64 tensor on {self.device}")
        ok_rows = (self.n_owned, self.n_rows) if rows is None else (rows,)
        if rows is not None or x.dim() == 3:
            if x.dim() != 3 or x.shape[1:] != (self.space.n_species, self.space.nb) \
                    or x.shape[0] not in ok_rows:
                raise ValueError(f"{name} has shape {tuple(x.shape)}, expected "
                                 f"(rows in {ok_rows}, {self.space.n_species}, "
                                 f"{self.space.nb})")

    def _ptr(self, x):
        return None if x is None else x.data_ptr()

    def rk_stage(self, U0, U, out, a: float, b: float, c: float, t: float = 0.0, acc=None):
        """out = a U0 + b U + c M^-1 L(U) in one fused pass.  The face sums
        accumulate in ``acc`` (default: ``out``), which must not alias U
        (nor U0 when a != 0)."""
        self._point_data_at(t, "rk_stage")
        self._check_vec("U", U, self.n_rows)
        self._check_vec("out", out)
        if U0 is not None:
            self._check_vec("U0", U0)
        if acc is not None:
            self._check_vec("acc", acc)
        self._call(self.lib.tdg_rk_stage, self._ctx, self._ptr(U0), U.data_ptr(),
                   out.data_ptr(), self._ptr(acc), float(a), float(b), float(c), float(t),
                   self._stream(), what="tdg_rk_stage")
        return out

    def rk_stage_part(self, U0, U, out, a: float, b: float, c: float, part: int,
                      t: float = 0.0, acc=None):
        """Half of ``rk_stage`` around a ghost exchange: part 1 = faces that
        read owned rows only, part 2 = the cut faces + the volume kernel
        (issue after the ghost rows of U are filled)."""
        self._check_vec("U", U, self.n_rows)
        self._check_vec("out", out)
        if U0 is not None:
            self._check_vec("U0", U0)
        if acc is not None:
            self._check_vec("acc", acc)
        self._call(self.lib.tdg_rk_stage_part, self._ctx, self._ptr(U0), U.data_ptr(),
                   out.data_ptr(), self._ptr(acc), float(a), float(b), float(c), float(t),
                   int(part), self._stream(), what="tdg_rk_stage_part")
        return out

    def _work_pair(self, work):
        if work is None:
            raise ValueError("ssprk3 needs two work vectors")
        if isinstance(work, (tuple, list)):
            w1, w2 = work
        else:
            if work.dim() != 4 or work.shape[0] != 2:
                raise ValueError("work must be a pair of state vectors or a (2, rows, S, nb) "
                                 "tensor")
            w1, w2 = work[0], work[1]
        self._check_vec("work[0]", w1, self.n_rows)
        self._check_vec("work[1]", w2, self.n_rows)
        return w1, w2

    def new_work(self):
        """The two SSP-RK3 work vectors (one (2, rows, S, nb) tensor)."""
        torch = _torch()
        return torch.empty((2, self.n_rows, self.space.n_species, self.space.nb),
                           dtype=torch.float64, device=self.device)

    def ssprk3_steps_host(self, U_host, nsteps: int, dt: float, t: float = 0.0,
                          U=None, work=None):
        """``nsteps`` SSP-RK3 steps of a pinned host state (CPU float64
        tensor of the U shape), with the state copied in and the result
        copied out every step (chunked copies overlapping the next step's
        copy-in and the last stage); ``U`` / ``work`` are the device state
        and work vectors (allocated here when not given).  Returns the
        (updated) host tensor; asynchronous on the current stream."""
        torch = _torch()
        shape = (self.n_rows, self.space.n_species, self.space.nb)
        if not isinstance(U_host, torch.Tensor) or U_host.device.type != "cpu" \
                or U_host.dtype != torch.float64 or tuple(U_host.shape) != shape \
                or not U_host.is_contiguous() or not U_host.is_pinned():
            raise ValueError(f"U_host must be a pinned, contiguous float64 CPU tensor {shape}")
        if U is None:
            U = torch.empty(shape, dtype=torch.float64, device=self.device)
        self._check_vec("U", U, self.n_rows)
        w1, w2 = self._work_pair(self.new_work() if work is None else work)
        self._call(self.lib.tdg_ssprk3_steps_host, self._ctx, U_host.data_ptr(), U.data_ptr(),
                   w1.data_ptr(), w2.data_ptr(), int(nsteps), float(t), float(dt),
                   self._stream(), what="tdg_ssprk3_steps_host")
        return U_host

    def ssprk3_step(self, U, work, dt: float, t: float = 0.0):
        """One Shu-Osher SSP-RK3 step in place on U (undecomposed meshes;
        slab runs use ``stepping.SSPRK3`` with the halo exchange).  ``work``
        = two work vectors (``new_work()``)."""
        if self._pd_t is not None and self._pd_model.time_dependent:
            # the three stages need the data at three times
            raise ValueError("time-dependent boundary data: step through apply / apply_f "
                             "(the reference's stepper call shape)")
        if self.n_rows != self.n_owned:
            raise ValueError("ssprk3_step needs an undecomposed mesh; use "
                             "stepping.SSPRK3(op, halo) for slab runs")
        self._check_vec("U", U, self.n_rows)
        w1, w2 = self._work_pair(work)
        self._call(self.lib.tdg_ssprk3_step, self._ctx, U.data_ptr(), w1.data_ptr(),
                   w2.data_ptr(), float(t), float(dt), self._stream(), what="tdg_ssprk3_step")
        return U

    def species_totals(self, U, out=None):
        """Device int u_s over the owned elements (reference
        ``fespace.py:170-174``); returns a CUDA tensor of S values."""
        torch = _torch()
        self._check_vec("U", U)
        if out is None:
            out = torch.empty(self.space.n_species, dtype=torch.float64, device=self.device)
        self._call(self.lib.tdg_species_totals, self._ctx, U.data_ptr(), out.data_ptr(),
                                                  self._stream(), what="tdg_species_totals")
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
        self._call(self.lib.tdg_species_l2, self._ctx, U.data_ptr(), None if V is None else V.data_ptr(), out.data_ptr(),
            self._stream(), what="tdg_species_l2")
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
        self._call(self.lib.tdg_mgs, self._ctx, V.data_ptr(), V.stride(0), int(j), w.data_ptr(),
                                       n, h.data_ptr(), self._stream(), what="tdg_mgs")
        return h

    def mgs_pass(self, V, i: int, j: int, w, h, n: int | None = None):
        """Pass i of the MGS sweep ending at j over the first ``n`` entries
        (slab runs: owned rows), leaving h[i] un-reduced across ranks (the
        caller all-reduces it before the next pass; the last pass leaves
        w . w)."""
        n = w.numel() if n is None else int(n)
        if V.dim() != 2 or not V.is_contiguous() or not w.is_contiguous():
            raise ValueError("mgs_pass needs a contiguous 2-D V and a contiguous w")
        if V.shape[1] < n or w.numel() < n or j + 1 > V.shape[0] or h.numel() < j + 2:
            raise ValueError("mgs_pass: inconsistent sizes")
        self._call(self.lib.tdg_mgs_pass, self._ctx, V.data_ptr(), V.stride(0), int(i), int(j),
                   w.data_ptr(), n, h.data_ptr(), self._stream(), what="tdg_mgs_pass")
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
        self._call(self.lib.tdg_scale_norm, self._ctx, w.data_ptr(), 0.0 if dev_div else float(hnext),
            hnext.data_ptr() if dev_div else None, v.data_ptr(), w.numel(), norm_out.data_ptr(),
            self._stream(), what="tdg_scale_norm")
        return v

    def jv_shift(self, U, v, vnorm, cnum: float, Up, eps_out):
        """eps = cnum / max(||v||, 1e-300) (device), Up = U + eps v
        (reference ``timeint.py:259-264``)."""
        n = U.numel()
        for name, x in (("U", U), ("v", v), ("Up", Up)):
            self._check_vec(name, x.reshape(-1))
        if v.numel() != n or Up.numel() != n:
            raise ValueError("jv_shift: size mismatch")
        self._call(self.lib.tdg_jv_shift, U.data_ptr(), v.data_ptr(), vnorm.data_ptr(),
                                            float(cnum), Up.data_ptr(), eps_out.data_ptr(), n,
                                            self._stream(), what="tdg_jv_shift")
        return Up

    def jv_diff(self, r, GU, eps):
        """r = (r - GU) / eps in place (device eps)."""
        self._check_vec("r", r.reshape(-1))
        self._check_vec("GU", GU.reshape(-1))
        if r.numel() != GU.numel():
            raise ValueError("jv_diff: size mismatch")
        self._call(self.lib.tdg_jv_diff, r.data_ptr(), GU.data_ptr(), eps.data_ptr(), r.numel(),
                                           self._stream(), what="tdg_jv_diff")
        return r

    def dot(self, x, y, out=None):
        x, y = x.reshape(-1), y.reshape(-1)
        self._check_vec("x", x)
        self._check_vec("y", y)
        if x.numel() != y.numel():
            raise ValueError("x and y differ in size")
        out = self._scalar[:1] if out is None else out
        self._call(self.lib.tdg_dot, self._ctx, x.data_ptr(), y.data_ptr(),
                                       x.numel(), out.data_ptr(), self._stream(), what="tdg_dot")
        return out

    def norm2(self, x, out=None):
        x = x.reshape(-1)
        self._check_vec("x", x)
        out = self._scalar[1:] if out is None else out
        self._call(self.lib.tdg_norm2, self._ctx, x.data_ptr(), x.numel(),
                                         out.data_ptr(), self._stream(), what="tdg_norm2")
        return out

    def axpby(self, a: float, x, b: float, y):
        if x.numel() != y.numel():
            raise ValueError("x and y differ in size")
        self._check_vec("x", x.reshape(-1))
        self._check_vec("y", y.reshape(-1))
        self._call(self.lib.tdg_axpby, float(a), x.data_ptr(), float(b),
                                         y.data_ptr(), x.numel(), self._stream(), what="tdg_axpby")
        return y

    def axpy_dev(self, s: float, alpha, x, y):
        if x.numel() != y.numel():
            raise ValueError("x and y differ in size")
        self._check_vec("x", x.reshape(-1))
        self._check_vec("y", y.reshape(-1))
        self._call(self.lib.tdg_axpy_dev, float(s), alpha.data_ptr(),
                                            x.data_ptr(), y.data_ptr(),
                                            x.numel(), self._stream(), what="tdg_axpy_dev")
        return y
