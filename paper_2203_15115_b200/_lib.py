"""ctypes binding of libtopovox_b200.so (the C-ABI in include/topovox_b200.h).

There is deliberately no fallback: if the library is missing, or no CUDA
device is visible, every compute entry point raises. The only host-side math
in this package is problem setup (mesh/selectors) and scalar driver logic.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import TopovoxError, raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtopovox_b200.so")

_lib = None

c_int, c_double, c_size_t, c_ll, P = ctypes.c_int, ctypes.c_double, ctypes.c_size_t, ctypes.c_longlong, ctypes.c_void_p


class CoarseND(ctypes.Structure):
    _fields_ = [
        ("n_levels", c_int), ("max_front", c_int), ("max_sep", c_int),
        ("d_meta", P), ("d_gmap", P), ("d_G", P), ("d_B", P),
        ("d_udof", P), ("d_fS", P), ("d_cU", P),
        ("d_fwd_items", P), ("d_bwd_items", P),
        ("h_fwd_ptr", P), ("h_bwd_ptr", P), ("h_fwd_wpr", P), ("h_bwd_wpr", P),
        ("h_split", P), ("d_asm_nodes", P), ("h_asm_ptr", P),
        ("n_top", c_int), ("top_off", ctypes.c_longlong), ("top_wpr", c_int),
        ("d_ZT", P), ("d_fT", P), ("d_tptr", P), ("d_tidx", P),
        ("d_perm", P),
        ("d_items", P), ("n_items", c_int), ("d_rel", P), ("d_cnt", P), ("d_ctl", P),
        ("d_factor", P), ("factor_bytes", c_size_t),
        ("fs_ld", ctypes.c_longlong), ("cu_ld", ctypes.c_longlong), ("ft_ld", ctypes.c_longlong),
        ("max_cols", c_int),
        ("top_tiles", c_int), ("d_tpart", P), ("tpart_ld", ctypes.c_longlong),
    ]


class FrontSet(ctypes.Structure):
    _fields_ = [
        ("d_fronts", P), ("d_pool", P), ("d_scratch", P), ("d_blocks", P), ("d_children", P), ("d_gmap", P),
        ("d_Es", P), ("mx", c_int), ("my", c_int), ("mz", c_int), ("d_err", P),
    ]


class PcgDesc(ctypes.Structure):
    _fields_ = [
        ("nx", c_int), ("ny", c_int), ("nz", c_int),
        ("h", c_double),
        ("h_mh45", P), ("h_kdiag3", P),
        ("d_occ", P), ("d_nflags", P), ("d_f", P), ("d_x", P),
        ("d_ws", P), ("ws_bytes", c_size_t),
        ("tol", c_double), ("max_iters", c_int), ("check_every", c_int),
        ("block", c_int), ("d_cen", P), ("d_S", P), ("d_keep", P),
        ("d_coarse", P), ("coarse_kind", c_int), ("coarse_nd", ctypes.POINTER(CoarseND)),
        ("projection", c_int), ("d_defl_nflags", P),
        ("iterations", c_int), ("residual", c_double), ("fnorm", c_double),
    ]


_SIGS = {
    "tvb_version": (c_int, []),
    "tvb_last_error": (ctypes.c_char_p, []),
    "tvb_modal_from_k0": (c_int, [P, P]),
    "tvb_matvec_ws_bytes": (c_size_t, [c_int, c_int, c_int]),
    "tvb_matvec": (c_int, [c_int, c_int, c_int, P, P, P, P, P, c_int, P, P, c_size_t, P]),
    "tvb_matvec_plan": (c_int, [c_int, c_int, c_int, P]),
    "tvb_matvec_host_ws_bytes": (c_size_t, [c_int, c_int, c_int]),
    "tvb_matvec_host": (c_int, [c_int, c_int, c_int, P, P, P, P, P, c_int, c_int, P, c_size_t, P]),
    "tvb_matvec_host_batch_ws_bytes": (c_size_t, [c_int, c_int, c_int]),
    "tvb_matvec_host_batch": (c_int, [c_int, c_int, c_int, P, c_int, P, P, P, P, c_int, c_int, P, c_size_t, P]),
    "tvb_fp64_peak_tflops": (c_double, [P]),
    "tvb_matvec_subset": (c_int, [c_int, c_int, c_int, P, P, P, P, c_ll, P, P, c_size_t, P]),
    "tvb_diag": (c_int, [c_int, c_int, c_int, P, P, P, P, c_int, P, P, P]),
    "tvb_node_flags": (c_int, [c_int, c_int, c_int, P, c_ll, P, P, P]),
    "tvb_reduce_ws_bytes": (c_size_t, [c_ll]),
    "tvb_dot": (c_int, [P, P, P, c_ll, P, P, c_size_t, P]),
    "tvb_defl_build": (c_int, [c_int, c_int, c_int, c_int, c_double, P, P, P, P, P, P]),
    "tvb_restrict": (c_int, [c_int, c_int, c_int, c_int, c_double, P, P, P, P, P, P, P]),
    "tvb_prolong": (c_int, [c_int, c_int, c_int, c_int, c_double, P, P, P, P, P, P, P, P]),
    "tvb_coarse_assemble_ws_bytes": (c_size_t, [c_int, c_int, c_int, c_int]),
    "tvb_coarse_assemble": (c_int, [c_int, c_int, c_int, c_int, c_double, P, P, P, P, P, P, P, P, c_size_t, P]),
    "tvb_coarse_dense": (c_int, [c_int, c_int, c_int, c_int, P, P, P]),
    "tvb_coarse_nd_solve": (c_int, [ctypes.POINTER(CoarseND), P, P, P]),
    "tvb_front_level": (c_int, [ctypes.POINTER(FrontSet), c_int, P, c_int, P, c_int, P, c_int, P]),
    "tvb_front_pack": (c_int, [ctypes.POINTER(FrontSet), c_int, P, P, c_ll, c_ll, P]),
    "tvb_front_pack_top": (c_int, [ctypes.POINTER(FrontSet), c_int, c_ll, c_int, P, P]),
    "tvb_pcg_ws_bytes": (c_size_t, [c_int, c_int, c_int, c_int]),
    "tvb_pcg_solve": (c_int, [ctypes.POINTER(PcgDesc), P]),
    "tvb_pcg_batch_ws_bytes": (c_size_t, [c_int, c_int, c_int, c_int, c_int]),
    "tvb_pcg_solve_batch": (c_int, [ctypes.POINTER(PcgDesc), c_int, P, P, P, P, P, P]),
    "tvb_elem_ws_bytes": (c_size_t, [c_int, c_int, c_int]),
    "tvb_element_state": (c_int, [c_int, c_int, c_int, c_double, c_double, c_double, P, P, P, P, P, P, c_int, P, P,
                                  c_size_t, P]),
    "tvb_adjoint_rhs": (c_int, [c_int, c_int, c_int, c_double, c_double, c_double, P, P, P, c_int, P, P, P, c_size_t,
                                P]),
    "tvb_sens_stress": (c_int, [c_int, c_int, c_int, c_double, c_double, c_double, P, P, P, P, P]),
    "tvb_maxabs": (c_int, [P, c_ll, P, P, c_size_t, P]),
    "tvb_combine": (c_int, [c_int, P, P, P, c_ll, P, P]),
    "tvb_select_ws_bytes": (c_size_t, [c_ll]),
    "tvb_threshold_select": (c_int, [P, P, c_ll, c_ll, c_double, c_double, P, P, c_size_t, P, P]),
    "tvb_threshold_select_ex": (c_int, [P, P, c_ll, c_ll, c_double, c_double, c_int, P, P, c_size_t, P, P]),
    "tvb_casting_project": (c_int, [c_int, c_int, c_int, c_int, c_int, P, P, P]),
    "tvb_nodal_block8": (c_int, [c_int, c_int, c_int, P, P, P, P]),
    "tvb_geo_matvec": (c_int, [c_int, c_int, c_int, P, P, P, P, P, c_int, c_double, P]),
    "tvb_lumped_mass": (c_int, [c_int, c_int, c_int, c_double, P, P, P]),
    "tvb_eigen_sens": (c_int, [c_int, c_int, c_int, c_double, c_double, c_double, P, P, c_double, P, P]),
    "tvb_buckling_sens": (c_int, [c_int, c_int, c_int, P, P, P, P, P, c_double, P, P]),
}

MASK_IN, MASK_OUT, ACCUMULATE = 1, 2, 4


def exported_symbols() -> list[str]:
    return list(_SIGS)


def lib():
    """Load (and type) the native library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TopovoxError(
                f"native library {LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    s = lib().tvb_last_error()
    return s.decode() if s else ""


def check(code: int, what: str) -> None:
    if code != 0:
        raise_for_status(code, what, last_error())


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise TopovoxError("no CUDA device visible: the topovox-b200 compute path runs only on the GPU")
    return torch


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr():
    import torch

    return torch.cuda.current_stream().cuda_stream


def host_array(a: np.ndarray):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.c_void_p)
