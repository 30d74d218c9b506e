"""ctypes binding of libmpgpu.so (include/mpgpu.h).

The product path has no CPU fallback: if the CUDA library is missing this module
raises on import, and every compute call fails loudly without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("MPGPU_LIB", Path(__file__).resolve().parent / "libmpgpu.so"))

if not LIB_PATH.exists():
    raise ImportError(
        f"libmpgpu.so not found at {LIB_PATH}: build it with "
        "`python paper_1410_1599_b200/build.py` (or __graft_entry__.build())")

lib = C.CDLL(str(LIB_PATH))

u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class MpgpuMat(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("prec", C.c_int32), ("nlimbs", C.c_int32),
                ("rec", vp), ("ld", C.c_int64), ("owned", C.c_int32)]


class MpgpuStats(C.Structure):
    _fields_ = [("mul", C.c_uint64), ("addsub", C.c_uint64), ("leaf_madds", C.c_uint64),
                ("device_ms", C.c_double), ("leaf_ms", C.c_double), ("preadd_ms", C.c_double),
                ("postadd_ms", C.c_double), ("launches", C.c_int32), ("depth", C.c_int32)]


MatP = C.POINTER(MpgpuMat)
StatsP = C.POINTER(MpgpuStats)

_SIGS = {
    "mpgpu_init": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "mpgpu_destroy": (None, [vp]),
    "mpgpu_last_error": (C.c_char_p, [vp]),
    "mpgpu_set_stream": (C.c_int, [vp, vp]),
    "mpgpu_get_stream": (vp, [vp]),
    "mpgpu_synchronize": (C.c_int, [vp]),
    "mpgpu_copy_device": (C.c_int, [vp, vp, vp, C.c_size_t]),
    "mpgpu_nlimbs_for": (C.c_int, [C.c_int32]),
    "mpgpu_record_words": (C.c_int, [C.c_int32]),
    "mpgpu_alloc_matrix": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int32, MatP]),
    "mpgpu_free_matrix": (C.c_int, [vp, MatP]),
    "mpgpu_upload": (C.c_int, [vp, MatP, vp, vp, vp, C.c_int32]),
    "mpgpu_download": (C.c_int, [vp, MatP, vp, vp, vp, C.c_int32]),
    "mpgpu_gemm": (C.c_int, [vp, C.c_int, C.c_int64, MatP, MatP, MatP, StatsP]),
    "mpgpu_gemm_host": (C.c_int, [vp, C.c_int, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_int64,
                                  vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int32, StatsP]),
    "mpgpu_fast_mul_trace": (C.c_int, [vp, C.c_int, C.c_int64, MatP, MatP, MatP, vp, C.POINTER(C.c_int)]),
    "mpgpu_addsub": (C.c_int, [vp, C.c_int, MatP, MatP, MatP]),
    "mpgpu_vec_op": (C.c_int, [vp, C.c_int, MatP, MatP, MatP]),
    "mpgpu_lu_blocked": (C.c_int, [vp, MatP, C.c_int64, C.c_int, C.c_int64, C.c_int, vp, i64p, StatsP]),
    "mpgpu_lu_blocked_host": (C.c_int, [vp, C.c_int32, C.c_int64, vp, vp, vp, C.c_int32, C.c_int64, C.c_int,
                                        C.c_int64, C.c_int, vp, i64p, StatsP]),
    "mpgpu_lu_solve": (C.c_int, [vp, MatP, vp, MatP, MatP, C.c_int, i64p]),
    "mpgpu_matrix_view": (C.c_int, [MatP, C.c_int64, C.c_int64, C.c_int64, C.c_int64, MatP]),
    "mpgpu_fast_plan": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, i64p]),
    "mpgpu_fast_leaves": (C.c_int, [vp, C.c_int, C.c_int64, MatP, MatP, C.c_int, C.c_int64, C.c_int64, vp,
                                    StatsP]),
    "mpgpu_fast_leaves_rows": (C.c_int, [vp, C.c_int, C.c_int64, MatP, MatP, C.c_int, C.c_int64, C.c_int64, vp,
                                         StatsP]),
    "mpgpu_malloc": (C.c_int, [vp, C.c_size_t, C.POINTER(vp)]),
    "mpgpu_free": (C.c_int, [vp, vp]),
    "mpgpu_ipc_handle": (C.c_int, [vp, vp, vp]),
    "mpgpu_ipc_open": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "mpgpu_ipc_close": (C.c_int, [vp, vp]),
    "mpgpu_fast_combine": (C.c_int, [vp, C.c_int, C.c_int64, C.c_int64, C.c_int, vp, MatP, StatsP]),
    "mpgpu_fast_combine_rows": (C.c_int, [vp, C.c_int, C.c_int64, C.c_int64, C.c_int, vp, C.c_int64, C.c_int64,
                                          MatP, StatsP]),
    "mpgpu_copy_device_2d": (C.c_int, [vp, vp, C.c_size_t, vp, C.c_size_t, C.c_size_t, C.c_size_t]),
    "mpgpu_count_fast": (C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, u64p]),
    "mpgpu_recursion_plan": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, i64p, C.c_int,
                                       C.POINTER(C.c_int)]),
    "mpgpu_gen": (C.c_int, [C.c_int, C.c_int64, C.c_uint64, C.c_int32, vp, vp, vp, C.c_int32]),
    "mpgpu_lu_solve_many": (C.c_int, [vp, MatP, vp, MatP, MatP, C.c_int, i64p]),
    "mpgpu_convert": (C.c_int, [vp, MatP, MatP]),
    "mpgpu_max_rel_error": (C.c_int, [vp, MatP, MatP, vp, vp, vp, i64p]),
    "mpgpu_solution_error": (C.c_int, [vp, MatP, MatP, vp, vp, vp, i64p]),
    "mpgpu_one_norm": (C.c_int, [vp, MatP, vp, vp, vp]),
    "mpgpu_choose_nmin": (C.c_int, [C.c_int, C.c_int32, C.c_int64, C.c_int64, C.c_int64, i64p,
                                    C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    "mpgpu_fast_owned_rows": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_int64,
                                        vp, C.c_int64, i64p]),
    "mpgpu_upload_strided": (C.c_int, [vp, MatP, vp, vp, vp, C.c_int32, C.c_int64]),
    "mpgpu_download_strided": (C.c_int, [vp, MatP, vp, vp, vp, C.c_int32, C.c_int64]),
    "mpgpu_group_init": (C.c_int, [C.c_uint32, C.POINTER(vp)]),
    "mpgpu_group_init_devices": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(vp)]),
    "mpgpu_group_destroy": (None, [vp]),
    "mpgpu_group_size": (C.c_int, [vp]),
    "mpgpu_group_device": (C.c_int, [vp, C.c_int]),
    "mpgpu_group_handle": (vp, [vp, C.c_int]),
    "mpgpu_group_last_error": (C.c_char_p, [vp]),
    "mpgpu_group_gemm_host": (C.c_int, [vp, C.c_int, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_int64,
                                        vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int32, StatsP]),
    "mpgpu_gemm_host_mask": (C.c_int, [C.c_uint32, C.c_int, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_int64,
                                       vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int32, StatsP, C.c_char_p,
                                       C.c_size_t]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)
