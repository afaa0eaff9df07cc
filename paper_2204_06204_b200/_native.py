"""ctypes binding of the C ABI in `include/bisimp_b200.h`.

This is the reference-side binding a maintainer of `bisimp` would add (see
INTEGRATION.md): the reference is pure Python, so its natural FFI for the
hot path is ctypes over plain pointers.  The library is built in-tree by
`paper_2204_06204_b200.build` into `paper_2204_06204_b200/lib/`.

There is no CPU fallback: if the library or a CUDA device is missing every
compute call raises `NativeUnavailable`.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libbisimp_b200.so")

BSP_OK, BSP_EINVAL, BSP_ENONFINITE, BSP_ECUDA, BSP_ENOMEM, BSP_EUNSUPPORTED, BSP_ESOLVE = range(7)
ALGO = {"fbto": 0, "pfbto_jacobi": 1, "cpfbto_krylov": 2, "pgd_exact": 3,
        "pcg_jacobi": 4, "mg_vcycle": 5, "mg_pcg": 6}


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a CUDA device) is not available: no fallback exists."""


class NativeError(RuntimeError):
    """A CUDA/runtime failure inside the native library."""


class SolverConfigC(C.Structure):
    """`bsp_solver_config` (include/bisimp_b200.h).  `struct_size` is the ABI
    version: the library reads only the first struct_size bytes and gives the
    optional trailing fields their defaults."""
    _fields_ = [
        ("struct_size", C.c_size_t),
        ("algorithm", C.c_int),
        ("eta", C.c_double),
        ("n_taps", C.c_int),
        ("taps", C.POINTER(C.c_double)),
        ("v_lo", C.c_double),
        ("v_hi", C.c_double),
        ("budget", C.c_double),
        ("beta", C.c_double),
        ("krylov_dim", C.c_int),
        ("tol_dv", C.c_double),
        ("tol_res", C.c_double),
        ("mean_projection", C.c_int),
        ("max_batch", C.c_int),
        ("inner_steps", C.c_int),
        ("mg_omega", C.c_double),
        ("mg_nu", C.c_int),
        ("mg_levels", C.c_int),
    ]

    def __init__(self, taps=None, **kw):
        super().__init__(**kw)
        self.struct_size = C.sizeof(SolverConfigC)
        if taps is not None:
            self.set_taps(taps)

    def set_taps(self, taps) -> None:
        import numpy as np
        # owned by the struct object until the library has copied it (create)
        self._taps = np.ascontiguousarray(taps, dtype=np.float64)
        self.n_taps = int(self._taps.size)
        self.taps = self._taps.ctypes.data_as(C.POINTER(C.c_double))


_P = C.c_void_p
_D = C.c_double
_I = C.c_int
_LL = C.c_longlong

# name -> argtypes (restype is int unless listed in _RESTYPE)
SIGNATURES = {
    "bsp_last_error": [],
    "bsp_version": [],
    "bsp_grid_create": [_I, _I, _P, _P, _P, C.POINTER(_P)],
    "bsp_grid_create_sparse": [_I, _I, _P, _LL, _P, _LL, _P, _P, C.POINTER(_P)],
    "bsp_grid_destroy": [_P],
    "bsp_grid_info": [_P, C.POINTER(_LL), C.POINTER(_LL), C.POINTER(_I)],
    "bsp_apply_stiffness": [_P, _P, _P, _P, _P],
    "bsp_apply_stiffness_premasked": [_P, _P, _P, _P, _P],
    "bsp_stiffness_diagonal": [_P, _P, _P, _P],
    "bsp_element_energies": [_P, _P, _P, _P],
    "bsp_residual": [_P, _P, _P, _P, _P, _P],
    "bsp_sensitivity": [_P, _P, _P, _D, _P, _I, _P, _P],
    "bsp_estimate_rho_max": [_P, _P, _P, _I, _P, _P],
    "bsp_estimate_sqjacobi_rho": [_P, _P, _P, _I, _P, _P],
    "bsp_krylov_apply": [_P, _P, _P, _I, _P, _P, _P],
    "bsp_low_level_step": [_P, _I, _P, _P, _D, _P, _I, _P, _P],
    "bsp_exact_solve": [_P, _P, _D, _P, _LL, _P, _P],
    "bsp_filter": [_P, _P, _P, _D, _I, _I, _P, _I, _I, _P],
    "bsp_mean_project": [_P, _LL, _P, _P],
    "bsp_project_simplex": [_P, _LL, _D, _D, _D, _P, _P],
    "bsp_high_level_step": [_P, _P, _LL, _D, _D, _D, _D, _P, _I, _P, _P],
    "bsp_density_frame": [_P, _LL, _P, _P],
    "bsp_density_pixels": [_P, _LL, _P, _P, _P],
    "bsp_standard_normal": [_P, _LL, _P, _P],
    "bsp_start_vector": [_P, _P, _P, _P],
    "bsp_mg_create": [_P, _I, C.POINTER(_P)],
    "bsp_mg_destroy": [_P],
    "bsp_mg_info": [_P, C.POINTER(_I), C.POINTER(_I)],
    "bsp_mg_level": [_P, _I, C.POINTER(_I), C.POINTER(_I), _P],
    "bsp_mg_setup": [_P, _P, _P],
    "bsp_mg_vcycle": [_P, _P, _P, _D, _I, _P],
    "bsp_pcg_apply": [_P, _P, _P, _P, _I, _D, _I, _P, _D, _P, _P],
    "bsp_nccl_unique_id": [_P, C.POINTER(_I)],
    "bsp_dist_slab_rows": [_I, _I, _I, _I, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I),
                           C.POINTER(_I)],
    "bsp_dist_create": [_I, _I, _I, _I, _P, _P, _P, _P, C.POINTER(SolverConfigC), _P, _D, _P,
                        C.POINTER(_P)],
    "bsp_dist_destroy": [_P],
    "bsp_dist_estimate_beta": [_P, _P, _I, C.POINTER(_D)],
    "bsp_dist_run": [_P, _LL, _I, _P, _P, C.POINTER(_I), C.POINTER(_I)],
    "bsp_dist_read": [_P, _I, _P],
    "bsp_dist_info": [_P, _P],
    "bsp_dist_comm_bench": [_P, _I, _P],
    "bsp_dist_stream": [_P],
    "bsp_solver_create": [_P, C.POINTER(SolverConfigC), _P, _P, C.POINTER(_P)],
    "bsp_solver_destroy": [_P],
    "bsp_solver_run": [_P, _LL, _I, _P, _P, C.POINTER(_I), C.POINTER(_I)],
    "bsp_solver_set_alphas": [_P, _LL, _I, _P],
    "bsp_solver_launch": [_P, _LL],
    "bsp_solver_finish": [_P, _LL, _I, _P, C.POINTER(_I), C.POINTER(_I)],
    "bsp_solver_read": [_P, _I, _P],
    "bsp_solver_read_state": [_P, _P, _P, _P, _P],
    "bsp_solver_read_frame": [_P, _I, _P],
    "bsp_solver_step_host": [_P, _LL, _D, _P, _P, _P, _P, _P],
    "bsp_solver_stamps": [_P, _I, _P],
    "bsp_device_clock": [_P, C.POINTER(_LL)],
    "bsp_solver_info": [_P, _P],
    "bsp_solver_stream": [_P],
}
_RESTYPE = {"bsp_last_error": C.c_char_p, "bsp_solver_stream": C.c_void_p,
            "bsp_dist_stream": C.c_void_p}

_lib = None
_lock = threading.Lock()


def lib_path() -> str:
    return _LIB_PATH


def load():
    """Load (once) and return the ctypes library handle; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise NativeUnavailable(
                f"{_LIB_PATH} is missing: build it with `python -m paper_2204_06204_b200.build` "
                "(the B200 path has no CPU fallback)")
        lib = C.CDLL(_LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, C.c_int)
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a C return code to the reference's exception classes."""
    if rc == BSP_OK:
        return
    msg = load().bsp_last_error().decode(errors="replace")
    if rc == BSP_EINVAL:
        raise ValueError(msg)
    if rc == BSP_ENONFINITE:
        from .solvers import DivergenceError
        raise DivergenceError(msg)
    if rc == BSP_ESOLVE:
        from .fea import LinearSolveError
        raise LinearSolveError(msg)
    if rc == BSP_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == BSP_ENOMEM:
        raise MemoryError(msg)
    raise NativeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
