"""ctypes binding of ``liblsgpu.so`` (the C ABI declared in ``include/lsgpu.h``).

The library is built in-tree (``paper_2601_05709_b200/liblsgpu.so``) by
``__graft_entry__.build()`` / ``make -C paper_2601_05709_b200/csrc``.  There is
no fallback: if the library is missing or no CUDA device is present, every
operation raises :class:`NativeUnavailable` -- the hot path never silently
drops to a CPU implementation.
"""

import ctypes
import os

import torch

from .errors import ConfigError, SolverError

LIB_PATH = os.environ.get("LSG_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblsgpu.so")

LSG_OK = 0
LSG_ERR_ARG = -1
LSG_ERR_CUDA = -2
LSG_ERR_NOCONV = -3
LSG_OP_ELASTICITY = 1
LSG_OP_H1 = 2
LSG_OP_PG_TRANSPORT = 3
LSG_OP_PG_REINIT = 4
LSG_OP_LAPLACE = 5

SCAL_FIELDS = ("atol", "rho", "alpha", "beta", "rr", "pq", "bb", "iters", "done", "zero_rhs",
               "maxiter", "first", "rz_new")
SCAL_DOUBLES = 16


class NativeUnavailable(RuntimeError):
    """liblsgpu.so could not be loaded or no CUDA device is available."""


class Grid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n", ctypes.c_int32 * 3),
                ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3)]


class Op(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad_", ctypes.c_int32), ("grid", Grid),
                ("words", ctypes.c_void_p), ("p", ctypes.c_double * 6),
                ("aux", ctypes.c_void_p * 4)]


class PcgWs(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("parity", ctypes.c_int32),
                ("x", ctypes.c_void_p), ("b", ctypes.c_void_p), ("r", ctypes.c_void_p),
                ("p", ctypes.c_void_p), ("q", ctypes.c_void_p), ("scal", ctypes.c_void_p),
                ("partials", ctypes.c_void_p), ("counters", ctypes.c_void_p),
                ("p_alt", ctypes.c_void_p), ("dinv", ctypes.c_void_p), ("p_ring", ctypes.c_void_p),
                ("r_alt", ctypes.c_void_p), ("q_alt", ctypes.c_void_p)]


_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int32
_G = ctypes.POINTER(Grid)
_O = ctypes.POINTER(Op)
_W = ctypes.POINTER(PcgWs)

# symbol -> (restype, argtypes); the full export list of include/lsgpu.h
SIGNATURES = {
    "lsg_abi_version": (ctypes.c_int32, []),
    "lsg_sizeof_op": (ctypes.c_int64, []),
    "lsg_sizeof_pcg_ws": (ctypes.c_int64, []),
    "lsg_sizeof_grid": (ctypes.c_int64, []),
    "lsg_last_error": (ctypes.c_char_p, []),
    "lsg_launch_count": (ctypes.c_int64, []),
    "lsg_num_nodes": (ctypes.c_int64, [_G]),
    "lsg_num_elements": (ctypes.c_int64, [_G]),
    "lsg_partials_per_rhs": (ctypes.c_int64, [_G]),
    "lsg_mesh_vertices": (ctypes.c_int, [_G, _P, _P]),
    "lsg_mesh_elements": (ctypes.c_int, [_G, _P, _P]),
    "lsg_material": (ctypes.c_int, [_G, _P, _P, _P, _P]),
    "lsg_indicator_quad": (ctypes.c_int, [_G, _P, _P, _P]),
    "lsg_h1_words": (ctypes.c_int, [_G, _P, _I, _P, _P]),
    "lsg_apply": (ctypes.c_int, [_O, _I, _P, _P, _P]),
    "lsg_diag": (ctypes.c_int, [_O, _P, _P]),
    "lsg_inv_diag": (ctypes.c_int, [_O, _P, _P]),
    "lsg_pcg_start": (ctypes.c_int, [_O, _W, _D, _D, _D, _P]),
    "lsg_pcg_iterate": (ctypes.c_int, [_O, _W, _I, _P]),
    "lsg_pcg_finish": (ctypes.c_int, [_O, _W, _P]),
    "lsg_graph_stats": (None, [_P]),
    "lsg_shape_rhs": (ctypes.c_int, [_O, _I, _P, _D, _P, _P, _P, _P, _P, _P, _P]),
    "lsg_heat_shape": (ctypes.c_int, [_O, _I, _P, _P, _P, _P, _D, _P, _P, _P, _P, _P, _P]),
    "lsg_inverse_misfit": (ctypes.c_int, [_G, _I, _P, _P, _P, _P, _P, _D, _D, _P, _P, _P, _P, _P, _P]),
    "lsg_inverse_tensors": (ctypes.c_int, [_G, _I, _P, _P, _P, _P, _P, _P, _P, _D, _D, _D, _D, _D,
                                           _P, _P, _P]),
    "lsg_strain_projection_rhs": (ctypes.c_int, [_G, _I, _P, _P, _P]),
    "lsg_s1_tensor": (ctypes.c_int, [_O, _I, _P, _P, _P, _P]),
    "lsg_tensor_rhs": (ctypes.c_int, [_G, _P, _P, _P, _P]),
    "lsg_velocity_rhs": (ctypes.c_int, [_O, _P, _P, _D, _P, _P]),
    "lsg_velocity_stats": (ctypes.c_int, [_O, _P, _P, _P, _P, _P, _P]),
    "lsg_transport": (ctypes.c_int, [_G, _P, _P, _D, _I, _I, _D, _P, _P, _P]),
    "lsg_reinit": (ctypes.c_int, [_G, _P, _D, _I, _D, _P, _P, _P, _P]),
    "lsg_cfl_speed": (ctypes.c_int, [_G, _P, _P, _P, _P, _P]),
    "lsg_pg_reinit_rhs": (ctypes.c_int, [_O, _P, _P]),
    "lsg_bicgstab_work_doubles": (ctypes.c_int64, [_G]),
    "lsg_bicgstab": (ctypes.c_int, [_O, _P, _P, _P, _D, _I, ctypes.POINTER(ctypes.c_int32),
                                    ctypes.POINTER(ctypes.c_double), _P]),
}

_lib = None


def load(require_device=True):
    """Load liblsgpu.so (once).  Raises NativeUnavailable when it cannot."""
    global _lib
    if require_device and not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing; build it with `make -C paper_2601_05709_b200/csrc`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        for name, struct in (("lsg_sizeof_op", Op), ("lsg_sizeof_grid", Grid),
                             ("lsg_sizeof_pcg_ws", PcgWs)):
            if getattr(lib, name)() != ctypes.sizeof(struct):
                raise NativeUnavailable(f"{LIB_PATH}: {name} = {getattr(lib, name)()} but the "
                                        f"ctypes mirror has {ctypes.sizeof(struct)} bytes")
        _lib = lib
    return _lib


def call(name, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != LSG_OK:
        msg = lib.lsg_last_error().decode(errors="replace")
        if rc == LSG_ERR_ARG:
            raise ConfigError(f"{name}: {msg}")
        if rc == LSG_ERR_NOCONV:
            raise SolverError(f"{name}: {msg}")
        raise RuntimeError(f"{name}: {msg}")
    return rc


def ptr(t):
    """Raw device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ConfigError("liblsgpu needs CUDA tensors")
    if not t.is_contiguous():
        raise ConfigError("liblsgpu needs contiguous tensors")
    return ctypes.c_void_p(t.data_ptr())


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def make_grid(dim, n, lo, hi):
    g = Grid()
    g.dim = dim
    for a in range(3):
        g.n[a] = int(n[a]) if a < dim else 0
        g.lo[a] = float(lo[a]) if a < dim else 0.0
        g.hi[a] = float(hi[a]) if a < dim else 1.0
    return g


def make_op(kind, grid, words, params, aux=()):
    op = Op()
    op.kind = kind
    op.grid = grid
    op.words = words.data_ptr() if words is not None else None
    for i in range(6):
        op.p[i] = float(params[i]) if i < len(params) else 0.0
    for i, t in enumerate(aux):
        op.aux[i] = t.data_ptr() if t is not None else None
    return op


__all__ = ["NativeUnavailable", "SolverError", "load", "call", "ptr", "stream", "make_grid",
           "make_op", "Grid", "Op", "PcgWs", "SIGNATURES", "LIB_PATH"]
