"""ctypes binding of the in-tree CUDA library ``libflowfem_b200.so`` (include/flowfem_b200.h).

The library is the product: there is no CPU fallback. Importing works without a GPU (so
the symbol table and the host-only partition code can be exercised on CPU); any call
that needs the device fails loudly when no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFB_LIB", os.path.join(HERE, "libflowfem_b200.so"))

MAX_SOLVES = 64


class RunConfigC(C.Structure):
    _fields_ = [("sigma", C.c_double), ("rho", C.c_double), ("alpha0", C.c_double),
                ("lambda0", C.c_double), ("illumination", C.c_int), ("parts", C.c_int),
                ("overlap", C.c_int), ("adapt", C.c_int), ("n_passes", C.c_int),
                ("kappa", C.c_double), ("eta_threshold", C.c_double), ("alpha_th", C.c_double),
                ("tol", C.c_double), ("max_iters", C.c_int)]


class RunStatsC(C.Structure):
    _fields_ = [("parts_x", C.c_int), ("parts_y", C.c_int), ("n_solves", C.c_int),
                ("iters", C.c_int * MAX_SOLVES), ("residual", C.c_double * MAX_SOLVES),
                ("eta_max", C.c_double * MAX_SOLVES), ("pcg_iterations", C.c_longlong),
                ("ms_terms", C.c_double), ("ms_factor", C.c_double), ("ms_pcg", C.c_double),
                ("ms_adapt", C.c_double), ("ms_total", C.c_double),
                ("factor_doubles", C.c_double), ("iter_bytes", C.c_double),
                ("ms_asm_per_iter", C.c_double), ("ms_factor_full", C.c_double),
                ("factor_flops", C.c_double)]


class SchwarzOptionsC(C.Structure):
    _fields_ = [("n_iters", C.c_int), ("workers", C.c_int), ("components", C.c_int),
                ("adapt", C.c_int), ("n_adapt", C.c_int), ("kappa", C.c_double),
                ("eta_threshold", C.c_double), ("alpha_th", C.c_double), ("method", C.c_int),
                ("cg_max_iters", C.c_int), ("cg_tolerance", C.c_double),
                ("record_alpha_history", C.c_int)]


class SchwarzStatsC(C.Structure):
    _fields_ = [("increments", C.c_void_p), ("seconds", C.c_void_p), ("eta_max", C.c_void_p),
                ("alpha_history", C.c_void_p), ("n_updates", C.c_int)]


_vp = C.c_void_p
_d = C.c_double
_i = C.c_int

# name -> (restype, argtypes); every symbol include/flowfem_b200.h declares
SIGNATURES = {
    "ffb_last_error": (C.c_char_p, []),
    "ffb_abi_version": (_i, []),
    "ffb_kernel_launches": (C.c_longlong, []),
    "ffb_create": (_i, [C.POINTER(_vp), _i]),
    "ffb_destroy": (_i, [_vp]),
    "ffb_set_stream": (_i, [_vp, _vp, _i]),
    "ffb_set_factor_storage": (_i, [_vp, _i]),
    "ffb_get_factor_storage": (_i, [_vp, C.POINTER(_i), C.POINTER(_i)]),
    "ffb_gaussian_smooth": (_i, [_vp, _i, _i, _vp, _d, _vp]),
    "ffb_compute_derivatives": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ffb_build_data_terms": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _d, _vp]),
    "ffb_frames_to_terms": (_i, [_vp, _i, _i, _vp, _vp, _d, _d, _vp]),
    "ffb_enumerate_splits": (_i, [_i, _i, _i, _vp, _vp, _vp, _i]),
    "ffb_choose_split": (_i, [_i, _i, _i, _vp, _vp, _vp]),
    "ffb_csr_spmv": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp]),
    "ffb_load_image": (_i, [C.c_char_p, _vp, _vp, _vp]),
    "ffb_save_pgm": (_i, [C.c_char_p, _i, _i, _vp]),
    "ffb_read_flo": (_i, [C.c_char_p, _vp, _vp, _vp, _vp]),
    "ffb_write_flo": (_i, [C.c_char_p, _i, _i, _vp, _vp]),
    "ffb_compute_metrics": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ffb_rcm_order": (_i, [_i, _i, _vp, _vp, _vp]),
    "ffb_csr_cg_solve": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _d, _i, _vp, _vp, _vp, _vp]),
    "ffb_csr_solve": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _i, _d, _i, _vp, _vp, _vp, _vp]),
    "ffb_build_partition": (C.c_long, [_i, _i, _i, _i, _i, _vp, C.c_long]),
    "ffb_assign_workers": (_i, [_i, _i, _vp]),
    "ffb_assemble_apply": (_i, [_vp, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp]),
    "ffb_error_indicator": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp]),
    "ffb_update_alpha": (_i, [_vp, _i, _vp, _vp, _d, _d, _d, _d, _vp]),
    "ffb_set_terms": (_i, [_vp, _i, _i, _vp]),
    "ffb_set_frames": (_i, [_vp, _i, _i, _vp, _vp, _d, _d]),
    "ffb_set_reg": (_i, [_vp, _vp, _vp]),
    "ffb_get_reg": (_i, [_vp, _vp, _vp]),
    "ffb_set_partition": (_i, [_vp, _i, _i, _i]),
    "ffb_pcg_solve": (_i, [_vp, _i, _d, _i, _i, _vp, _vp, _vp]),
    "ffb_adapt": (_i, [_vp, _i, _d, _d, _d, _vp]),
    "ffb_schwarz_solve": (_i, [_vp, _i, _i, _i, _i, _d, _d, _d, _i, _vp, _vp, _vp]),
    "ffb_schwarz_run": (_i, [_vp, C.POINTER(SchwarzOptionsC), _vp, C.POINTER(SchwarzStatsC)]),
    "ffb_energy": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _i, _vp]),
    "ffb_energy_resident": (_i, [_vp, _i, _vp]),
    "ffb_assemble_system": (_i, [_vp, _i, _i, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp,
                                 _vp, _vp, _vp, _vp, _vp]),
    "ffb_chol_create": (_i, [_vp, C.POINTER(_vp)]),
    "ffb_chol_destroy": (_i, [_vp]),
    "ffb_chol_analyze": (_i, [_vp, _i, _i, _vp, _vp]),
    "ffb_chol_factorize": (_i, [_vp, _i, _vp]),
    "ffb_chol_solve": (_i, [_vp, _i, _vp, _vp]),
    "ffb_chol_info": (_i, [_vp, _vp, _vp]),
    "ffb_set_partition_flat": (_i, [_vp, _vp, C.c_long]),
    "ffb_comm_nccl_id": (_i, [_vp]),
    "ffb_comm_init_nccl": (_i, [_vp, _i, _i, _vp]),
    "ffb_comm_local_hub": (_i, [_i, C.POINTER(_vp)]),
    "ffb_comm_local_hub_destroy": (_i, [_vp]),
    "ffb_comm_init_local": (_i, [_vp, _vp, _i]),
    "ffb_comm_info": (_i, [_vp, _vp, _vp, _vp]),
    "ffb_comm_rows": (_i, [_i, _i, _i, _i, _i, _i, _i, _vp]),
    "ffb_run_on_frames": (_i, [_vp, _i, _i, _vp, _vp, C.POINTER(RunConfigC), _vp, _vp,
                               C.POINTER(RunStatsC)]),
    "ffb_run_on_frames_dev": (_i, [_vp, _i, _i, _vp, _vp, C.POINTER(RunConfigC), _vp,
                                   C.POINTER(RunStatsC)]),
}

_lib = None


def load():
    """Load and type the library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"flowfem_b200: {LIB_PATH} is missing; run `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().ffb_last_error().decode(errors="replace")
