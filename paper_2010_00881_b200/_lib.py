"""ctypes binding of libfcm_mg.so (include/fcm_mg.h).  Argument marshalling only.

The library must exist: there is no CPU fallback.  A missing or stale build raises."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfcm_mg.so")

FCM_OK = 0
FCM_NOT_CONVERGED = 1
ERRORS = {-1: "FCM_EINVAL", -2: "FCM_ENOMEM", -3: "FCM_ESINGULAR", -4: "FCM_EINDEF",
          -5: "FCM_ECUDA", -6: "FCM_ENCCL"}


class FcmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n", C.c_int32 * 3), ("h", C.c_double), ("p", C.c_int32),
                ("space", C.c_int32), ("n_f", C.c_int32), ("dirichlet_faces", C.c_uint32)]


class Params(C.Structure):
    _fields_ = [("block", C.c_int32), ("omega", C.c_double), ("n_pre", C.c_int32),
                ("n_post", C.c_int32), ("coarse", C.c_int32), ("coarse_rtol", C.c_double),
                ("coarse_maxit", C.c_int32), ("stream", C.c_void_p)]


class Slab(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("z_begin", C.c_int32), ("z_end", C.c_int32),
                ("nccl_id", C.c_void_p)]


class Physics(C.Structure):
    _fields_ = [("kind", C.c_int32), ("alpha", C.c_double), ("E", C.c_double), ("nu", C.c_double),
                ("depth", C.c_int32), ("traction_face", C.c_int32)]


class HpSpec(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n", C.c_int32), ("p", C.c_int32), ("kmax", C.c_int32),
                ("refine", C.c_int32), ("dirichlet_faces", C.c_uint32), ("phys", Physics),
                ("n_voids", C.c_int64), ("centres", C.c_void_p), ("radii", C.c_void_p)]


_lib = None

P = C.c_void_p
D = C.c_double
I32 = C.c_int32
I64 = C.c_int64
_SIGS = {
    "fcm_element_size": (I32, [P]),
    "fcm_gen_classify": (I32, [P, I64, P, P, P, P]),
    "fcm_gen_element_matrices": (I32, [P, P, I64, P, P, P, P, I64, P, P, P, P, I32]),
    "fcm_mg_setup": (I32, [P, P, P, P, D, I64, P, P, P]),
    "fcm_mg_destroy": (I32, [P]),
    "fcm_mg_nlevels": (I32, [P, P]),
    "fcm_mg_ndofs": (I32, [P, I32, P]),
    "fcm_mg_level_m": (I32, [P, I32, P]),
    "fcm_mg_block_counts": (I32, [P, I32, P, P]),
    "fcm_mg_lowrank_info": (I32, [P, I32, P, P]),
    "fcm_gen_cut_matrices_device": (I32, [P, P, C.c_int64, P, P, C.c_int64, P, P, P]),
    "fcm_mg_export_block_inverses": (I32, [P, I32, P, P, P, P, P]),
    "fcm_mg_dof_keys": (I32, [P, P]),
    "fcm_mg_load": (I32, [P, P, P, P, I32, P]),
    "fcm_apply": (I32, [P, I32, P, P]),
    "fcm_mg_smooth": (I32, [P, I32, P, P]),
    "fcm_mg_smooth_part": (I32, [P, I32, I32, P, P]),
    "fcm_mg_coarse_solve": (I32, [P, P, P, P]),
    "fcm_mg_vcycle": (I32, [P, P, P]),
    "fcm_pcg_solve": (I32, [P, P, P, D, I32, P, P]),
    "fcm_pcg_solve_host": (I32, [P, P, P, D, I32, P, P]),
    "fcm_mg_solve": (I32, [P, P, P, D, I32, P, P]),
    "fcm_mg_stats": (I32, [P, P, P]),
    "fcm_mg_coarse_info": (I32, [P, P, P, P]),
    "fcm_slab_bounds": (I32, [I32, I32, I32, P, P]),
    "fcm_slab_layout": (I32, [P, I32, I32, I32, P, P, P, P, P, P, P]),
    "fcm_slab_coarse_map": (I32, [P, I32, I32, P, P]),
    "fcm_nccl_unique_id": (I32, [P]),
    "fcm_mg_setup_slab": (I32, [P, P, P, P, P, D, I64, P, P, I64, P, P, P]),
    "fcm_mg_launch_count": (I32, [P, P]),
    "fcm_hp_generate": (I32, [P, P]),
    "fcm_hp_disc_destroy": (I32, [P]),
    "fcm_hp_disc_info": (I32, [P, P, P, P, P, P]),
    "fcm_hp_disc_levels": (I32, [P, P, P, P]),
    "fcm_hp_disc_keys": (I32, [P, P]),
    "fcm_hp_disc_load": (I32, [P, P]),
    "fcm_hp_disc_leaves": (I32, [P, P, P, P, P]),
    "fcm_hp_setup": (I32, [P, P, P]),
    "fcm_hp_destroy": (I32, [P]),
    "fcm_hp_apply": (I32, [P, I32, P, P]),
    "fcm_hp_smooth": (I32, [P, I32, P, P]),
    "fcm_hp_time_smooth": (I32, [P, I32, P, P, I32, P]),
    "fcm_hp_vcycle": (I32, [P, P, P]),
    "fcm_hp_pcg_solve": (I32, [P, P, P, D, I32, P, P]),
    "fcm_hp_mg_solve": (I32, [P, P, P, D, I32, P, P]),
    "fcm_hp_export_blocks": (I32, [P, I32, P, P, P, P, P, P]),
    "fcm_hp_stats": (I32, [P, P, P, P]),
    "fcm_last_error": (C.c_char_p, []),
}
EXPORTED = tuple(_SIGS)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2010_00881_b200.build` "
                              "(the CUDA path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc, allow_not_converged=False):
    if rc == FCM_OK or (allow_not_converged and rc == FCM_NOT_CONVERGED):
        return rc
    msg = lib().fcm_last_error().decode()
    raise FcmError(rc, msg)
