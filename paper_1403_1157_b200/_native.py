"""ctypes binding of ``libtaxisdg_b200.so`` (C-ABI: include/taxisdg_b200.h).

The library is built in-tree by ``paper_1403_1157_b200.build``.  There is
no fallback: if the library is missing or fails to load, importing the
operator raises -- the product path never silently runs on the CPU.
"""

from __future__ import annotations

import ctypes
import os

from .build import LIB

__all__ = ["lib", "TdgDesc", "check", "TDG_OK", "load"]

TDG_OK, TDG_E_INVALID, TDG_E_UNSUPPORTED, TDG_E_CUDA = 0, -1, -2, -3
ABI_VERSION = 9

_p = ctypes.c_void_p
_d = ctypes.c_double
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64


class TdgDesc(ctypes.Structure):
    _fields_ = [
        ("dim", _i32), ("order", _i32), ("n_species", _i32), ("nb", _i32),
        ("nq_vol", _i32), ("nq_face", _i32), ("model", _i32), ("scheme", _i32),
        ("n_elements", _i64), ("n_ghost", _i64), ("n_int_faces", _i64),
        ("n_bnd_faces", _i64),
        ("chi_e", _d), ("adj_sign", _d), ("ip_eta", _d),
        ("diffusivity", _p), ("lin_source", _p), ("params", _p),
        ("vol_phi", _p), ("vol_grad", _p), ("vol_w", _p), ("vol_stiff", _p),
        ("face_B", _p), ("face_G", _p), ("face_Pw", _p), ("face_w", _p),
        ("elem_geo", _p),
        ("if_elems", _p), ("if_code", _p), ("if_geo", _p),
        ("bf_elem", _p), ("bf_code", _p), ("bf_geo", _p),
        ("face_mma", _p), ("vol_tc", _p),
        ("face_tc", _p), ("face_blocks", _p), ("n_face_blocks", _i64),
        ("face_tc_fold", _p), ("if_fold", _p),
        ("face_groups", _p), ("n_face_groups", _i64), ("face_modal", _p),
        ("if_bval", _p), ("bf_qval", _p),
        ("seg_chunk_ptr", _p), ("if_code_add", _p), ("bf_code_add", _p),
        ("vol_cls_tab", _p), ("vol_perm", _p), ("vol_task_cls", _p), ("n_vol_tasks", _i64),
        ("vol_chunk_tasks", _p),
        ("n_segments", _i32), ("n_segments_cut", _i32), ("seg_ptr", _p),
    ]


_lib = None


def load(path: str = LIB):
    global _lib
    if _lib is not None:
        return _lib
    # A/B timing of alternative builds (tools/): TDG_LIB names another
    # in-tree build of the same library
    path = os.environ.get("TDG_LIB", path)
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m "
            "paper_1403_1157_b200.build` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    lib.tdg_version.restype = ctypes.c_int
    lib.tdg_last_error.restype = ctypes.c_char_p
    lib.tdg_create.argtypes = [ctypes.POINTER(TdgDesc), ctypes.POINTER(_p)]
    lib.tdg_destroy.argtypes = [_p]
    lib.tdg_apply.argtypes = [_p, _p, _p, _d, ctypes.c_int, _p]
    lib.tdg_rk_stage.argtypes = [_p, _p, _p, _p, _p, _d, _d, _d, _d, _p]
    lib.tdg_species_totals.argtypes = [_p, _p, _p, _p]
    lib.tdg_ssprk3_steps_host.argtypes = [_p, _p, _p, _p, _p, _i64, _d, _d, _p]
    lib.tdg_apply_host.argtypes = [_p, _p, _p, _p, _p, _d, ctypes.c_int, _p]
    lib.tdg_species_l2.argtypes = [_p, _p, _p, _p, _p]
    lib.tdg_mgs.argtypes = [_p, _p, _i64, ctypes.c_int, _p, _i64, _p, _p]
    lib.tdg_mgs_pass.argtypes = [_p, _p, _i64, ctypes.c_int, ctypes.c_int, _p, _i64, _p, _p]
    lib.tdg_rk_stage_part.argtypes = [_p, _p, _p, _p, _p, _d, _d, _d, _d, ctypes.c_int, _p]
    lib.tdg_ssprk3_step.argtypes = [_p, _p, _p, _p, _d, _d, _p]
    lib.tdg_color_faces.argtypes = [_i64, _p, _p, _i64, _p, _p]
    lib.tdg_dot.argtypes = [_p, _p, _p, _i64, _p, _p]
    lib.tdg_norm2.argtypes = [_p, _p, _i64, _p, _p]
    lib.tdg_axpby.argtypes = [_d, _p, _d, _p, _i64, _p]
    lib.tdg_axpy_dev.argtypes = [_d, _p, _p, _p, _i64, _p]
    lib.tdg_scale_norm.argtypes = [_p, _p, _d, _p, _p, _i64, _p, _p]
    lib.tdg_jv_shift.argtypes = [_p, _p, _p, _d, _p, _p, _i64, _p]
    lib.tdg_jv_diff.argtypes = [_p, _p, _p, _i64, _p]
    lib.tdg_profile.argtypes = [_p, ctypes.c_int]
    lib.tdg_set_variant.argtypes = [_p, ctypes.c_int]
    lib.tdg_profile_read.argtypes = [_p, ctypes.POINTER(_d), ctypes.POINTER(_i64)]
    lib.tdg_face_runs.argtypes = [_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
    lib.tdg_fp64_probe.argtypes = [_p, _i64, _p]
    lib.tdg_fp64_probe_threads.restype = _i64
    lib.tdg_dmma_probe.argtypes = [_p, _i64, _p]
    for name in ("tdg_face_runs", "tdg_apply_host", "tdg_mgs_pass", "tdg_color_faces", "tdg_ssprk3_steps_host", "tdg_species_l2", "tdg_mgs", "tdg_species_totals", "tdg_rk_stage_part", "tdg_dmma_probe", "tdg_set_variant", "tdg_profile", "tdg_profile_read", "tdg_fp64_probe",
                 "tdg_create", "tdg_destroy", "tdg_apply", "tdg_rk_stage",
                 "tdg_ssprk3_step", "tdg_dot", "tdg_norm2", "tdg_axpby",
                 "tdg_axpy_dev", "tdg_scale_norm", "tdg_jv_shift", "tdg_jv_diff"):
        getattr(lib, name).restype = ctypes.c_int
    if lib.tdg_version() != ABI_VERSION:
        raise ImportError("libtaxisdg_b200.so ABI version mismatch; rebuild")
    _lib = lib
    return lib


def lib():
    return load()


def check(rc: int, what: str = "tdg call") -> None:
    if rc == TDG_OK:
        return
    msg = _lib.tdg_last_error().decode() if _lib is not None else "?"
    if rc in (TDG_E_INVALID, TDG_E_UNSUPPORTED):
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")
