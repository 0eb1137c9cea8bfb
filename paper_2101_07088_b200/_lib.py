"""ctypes binding of libslabewald_cuda.so (include/slabewald.h).

The library is built in-tree (``_build.py``); there is no fallback: if it
cannot be loaded the solver raises.  Structures mirror the C declarations
field for field.
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libslabewald_cuda.so")

SE_OK = 0
SE_ERR_VALUE, SE_ERR_FLOAT, SE_ERR_LINALG, SE_ERR_CUDA, SE_ERR_MEMORY = \
    1, 2, 3, 4, 5

NEED_ENERGY = 1 << 0
NEED_FORCES = 1 << 1
NEED_POTENTIAL = 1 << 2
SUBTRACT_SELF = 1 << 3
CORRECTION = 1 << 4
FORCE_GENERAL = 1 << 5
TIMINGS = 1 << 6
FP32 = 1 << 7
PAIR_HASH = 1 << 8
GRAPH = 1 << 9

#: every entry point declared in include/slabewald.h
EXPORTS = ("se_plan_create", "se_plan_destroy", "se_plan_set_stream",
           "se_set_charges", "se_solve",
           "se_solve_device", "se_near_field", "se_build_partition",
           "se_debug_fetch", "se_fp64_peak", "se_last_error", "se_version",
           "se_shard_spread", "se_shard_fields", "se_shard_charges",
           "se_dist_setup", "se_dist_buffers", "se_dist_forward",
           "se_dist_modes", "se_dist_fields", "se_steric_forces",
           "se_tp_create", "se_tp_destroy", "se_tp_set_stream", "se_tp_set_graph", "se_tp_poisson",
           "se_tp_forces", "se_tp_forces_device", "se_steric_forces_device",
           "se_bd_first_noise_device", "se_bd_step_device", "se_shard_spread_own",
           "se_shard_near", "se_shard_charges_own")


class SeBdParams(ctypes.Structure):
    """se_bd_params (include/slabewald.h)."""
    _fields_ = [(n, ctypes.c_double) for n in (
        "dt", "mu", "kT", "max_disp", "z_lo", "z_hi", "Lx", "Ly", "H", "a", "U0", "r_m")] + \
        [(n, ctypes.c_int32) for n in ("p", "wall", "has_zb", "max_retries")] + \
        [("seed", ctypes.c_uint64)]


class SeParams(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in (
        "Lx", "Ly", "H", "eps", "eps_b", "eps_t", "g_w", "xi", "g_t", "H_E",
        "r_nf", "r_cut", "k_max", "z0", "z1", "xi_is_inf")] + \
        [(n, ctypes.c_int32) for n in ("Nx", "Ny", "Nz", "refine")]


class SeDiag(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in (
        "ai1", "ai2", "discrepancy", "B_i", "A_i", "A_b", "A_t",
        "psi_i_bottom", "psi_i_top", "psi_b_bottom", "psi_t_top",
        "U_wall")] + [
        ("warn_discrepancy", ctypes.c_int32), ("n_sources", ctypes.c_int32),
        ("n_pairs", ctypes.c_int64), ("n_launches", ctypes.c_int64),
        ("t_ms", ctypes.c_double * 16)]


_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64
_I64P = ctypes.POINTER(ctypes.c_int64)
_I32P = ctypes.POINTER(ctypes.c_int32)

_lib = None


def load():
    """Load (once) and return the library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            "libslabewald_cuda.so is not built (%s); run "
            "`python -m paper_2101_07088_b200._build`" % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    lib.se_plan_create.argtypes = [ctypes.POINTER(SeParams), _D, _D, _D, _D,
                                   _D, _D, _D, _D, ctypes.c_int,
                                   ctypes.POINTER(_P)]
    lib.se_plan_create.restype = ctypes.c_int
    lib.se_plan_destroy.argtypes = [_P]
    lib.se_plan_destroy.restype = None
    lib.se_plan_set_stream.argtypes = [_P, ctypes.c_void_p]
    lib.se_plan_set_stream.restype = ctypes.c_int
    lib.se_set_charges.argtypes = [_P, _D, _I64]
    lib.se_set_charges.restype = ctypes.c_int
    lib.se_solve.argtypes = [_P, _D, _I64, ctypes.c_uint32, _D, _D, _D,
                             ctypes.POINTER(SeDiag)]
    lib.se_solve.restype = ctypes.c_int
    lib.se_solve_device.argtypes = [_P, ctypes.c_void_p, _I64,
                                    ctypes.c_uint32, ctypes.c_void_p,
                                    ctypes.c_void_p, _D,
                                    ctypes.POINTER(SeDiag)]
    lib.se_solve_device.restype = ctypes.c_int
    lib.se_near_field.argtypes = [ctypes.POINTER(SeParams), ctypes.c_int, _D,
                                  _D, _I64, _D, _I64, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, _D, _D]
    lib.se_near_field.restype = ctypes.c_int
    lib.se_build_partition.argtypes = [ctypes.POINTER(SeParams), ctypes.c_int,
                                       _D, _D, _I64, _I64P, _I64P, _I64P,
                                       _I64P, _I64P, _D, _D, _I64P, _I32P]
    lib.se_build_partition.restype = ctypes.c_int
    lib.se_debug_fetch.argtypes = [_P, ctypes.c_int, ctypes.c_void_p, _I64]
    lib.se_debug_fetch.restype = ctypes.c_int64
    lib.se_shard_spread.argtypes = [_P, ctypes.c_void_p, _I64, _I64, _I64,
                                    ctypes.c_uint32,
                                    ctypes.POINTER(ctypes.c_void_p), _I64P]
    lib.se_shard_spread.restype = ctypes.c_int
    lib.se_shard_fields.argtypes = [_P]
    lib.se_shard_fields.restype = ctypes.c_int
    lib.se_shard_charges.argtypes = [_P, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, _D, ctypes.POINTER(SeDiag)]
    lib.se_shard_charges.restype = ctypes.c_int
    _v = ctypes.c_void_p
    lib.se_shard_spread_own.argtypes = [_P, _v, _I64, _I64, _I64, ctypes.c_uint32,
                                        ctypes.POINTER(ctypes.c_void_p), _I64P]
    lib.se_shard_spread_own.restype = ctypes.c_int
    lib.se_shard_near.argtypes = [_P, _v, _v, _v, _I64, _I64, ctypes.c_int, _v, _v, _v, _v]
    lib.se_shard_near.restype = ctypes.c_int
    lib.se_shard_charges_own.argtypes = [_P, _v, _v, _v, _v, _v, _D, ctypes.POINTER(SeDiag)]
    lib.se_shard_charges_own.restype = ctypes.c_int
    lib.se_dist_setup.argtypes = [_P, ctypes.c_int, ctypes.c_int, _I64P]
    lib.se_dist_setup.restype = ctypes.c_int
    lib.se_dist_buffers.argtypes = [_P, ctypes.POINTER(ctypes.c_void_p)]
    lib.se_dist_buffers.restype = ctypes.c_int
    for name in ("se_dist_forward", "se_dist_modes", "se_dist_fields"):
        getattr(lib, name).argtypes = [_P]
        getattr(lib, name).restype = ctypes.c_int
    _f = ctypes.c_double
    lib.se_steric_forces.argtypes = [ctypes.c_int, _D, _I64, _f, _f, _f, _f, _f, _f,
                                     ctypes.c_int, _D]
    lib.se_steric_forces.restype = ctypes.c_int
    lib.se_tp_create.argtypes = [ctypes.c_int, _f, _f, _f, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, _f, ctypes.POINTER(ctypes.c_void_p)]
    lib.se_tp_destroy.argtypes = [ctypes.c_void_p]
    lib.se_tp_set_stream.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.se_tp_set_graph.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.se_tp_poisson.argtypes = [ctypes.c_void_p, _D, ctypes.c_int, _D, _D]
    lib.se_tp_forces.argtypes = [ctypes.c_void_p, _D, _D, _I64, _f, _f, _f, _f, _f, _D]
    lib.se_tp_forces_device.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        _I64, _f, _f, _f, _f, _f, ctypes.c_void_p]
    _v = ctypes.c_void_p
    lib.se_steric_forces_device.argtypes = [ctypes.c_int, _v, _v, _I64, _f, _f, _f, _f, _f, _f,
                                            _f, _f, ctypes.c_int, _v]
    lib.se_bd_first_noise_device.argtypes = [ctypes.c_int, _v, _I64, ctypes.c_uint64, _v]
    lib.se_bd_step_device.argtypes = [ctypes.c_int, _v, _v, _v, _v, _v, _v, _I64,
                                      ctypes.POINTER(SeBdParams),
                                      ctypes.POINTER(ctypes.c_uint64),
                                      ctypes.POINTER(ctypes.c_int64)]
    for name in ("se_steric_forces_device", "se_bd_first_noise_device", "se_bd_step_device"):
        getattr(lib, name).restype = ctypes.c_int
    for name in ("se_tp_create", "se_tp_destroy", "se_tp_set_stream", "se_tp_set_graph",
                 "se_tp_poisson", "se_tp_forces", "se_tp_forces_device", "se_steric_forces_device",
           "se_bd_first_noise_device", "se_bd_step_device", "se_shard_spread_own",
           "se_shard_near", "se_shard_charges_own"):
        getattr(lib, name).restype = ctypes.c_int
    lib.se_fp64_peak.argtypes = [ctypes.c_int, _D]
    lib.se_fp64_peak.restype = ctypes.c_int
    lib.se_last_error.argtypes = []
    lib.se_last_error.restype = ctypes.c_char_p
    lib.se_version.argtypes = []
    lib.se_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(code):
    """Map a library error code to the reference's exception type."""
    if code == SE_OK:
        return
    msg = load().se_last_error().decode()
    if code == SE_ERR_VALUE:
        raise ValueError(msg)
    if code == SE_ERR_FLOAT:
        raise FloatingPointError(msg)
    if code == SE_ERR_LINALG:
        raise np.linalg.LinAlgError(msg)
    if code == SE_ERR_MEMORY:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def dptr(a):
    """double* of a C-contiguous float64 array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_D)


def as_f64(a, shape=None):
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        out = out.reshape(shape)
    return out


def params_struct(geometry, params, refine=1):
    xi_inf = bool(np.isinf(params.xi))
    return SeParams(
        Lx=geometry.Lx, Ly=geometry.Ly, H=geometry.H, eps=geometry.eps,
        eps_b=geometry.eps_b, eps_t=geometry.eps_t, g_w=params.g_w,
        xi=float(params.xi), g_t=params.g_t, H_E=params.H_E,
        r_nf=params.r_nf, r_cut=params.r_cut, k_max=params.k_max,
        z0=params.z0, z1=params.z1, xi_is_inf=1.0 if xi_inf else 0.0,
        Nx=int(params.Nx), Ny=int(params.Ny), Nz=int(params.Nz),
        refine=int(refine))
