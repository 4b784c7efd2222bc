"""ctypes binding of librwb.so, the C ABI declared in include/rwb.h.

There is no CPU fallback: importing works anywhere (so the host logic can be
tested on machines without a GPU), but every call into the library raises
`NativeUnavailable` when the shared library is missing, and the first call
checks that a Blackwell (sm_100) device is current.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.environ.get("RWB_LIBRARY") or os.path.join(LIB_DIR, "librwb.so")  # RWB_LIBRARY: diagnostics builds

c_int32, c_int64, c_float, c_void_p, c_size_t = (
    ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t)

ABI_VERSION = 2
SOLVE_NO_GRAPH = 1
SOLVE_STREAMING = 2
SOLVE_NO_COOP = 4
SOLVE_CLUSTER16 = 8
SOLVE_SPLIT_Z = 16
SOLVE_SETUP2 = 32
SOLVE_SETUP_ONLY = 128
SOLVE_NO_SETUP = 256
SOLVE_STATS_DEVICE = 512
SOLVE_CLUSTER4 = 1024
SOLVE_NO_MG = 2048
SOLVE_NO_COARSE = 4096
SOLVE_MG = 8192
PATH_STREAMING, PATH_RESIDENT, PATH_COOPERATIVE, PATH_MULTIGRID = 0, 1, 2, 3

# every symbol include/rwb.h declares, with (restype, argtypes)
SIGNATURES = {
    "rwb_abi_version": (c_int32, []),
    "rwb_last_error": (ctypes.c_char_p, []),
    "rwb_kernel_launches": (c_int64, []),
    "rwb_device_info": (c_int32, [ctypes.POINTER(c_int32)] * 3),
    "rwb_lod_down_f32": (c_int32, [c_int32, ctypes.POINTER(c_int64), c_void_p, c_void_p, c_void_p]),
    "rwb_project_seeds_u8": (c_int32, [c_int32, ctypes.POINTER(c_int64), c_void_p, c_void_p, c_void_p]),
    "rwb_upsample_f32": (c_int32, [c_int32, ctypes.POINTER(c_int64), c_void_p, ctypes.POINTER(c_int64),
                                   c_void_p, c_void_p]),
    "rwb_upsample_window_f32": (c_int32, [c_int32] + [ctypes.POINTER(c_int64)] * 3 + [c_void_p] +
                                [ctypes.POINTER(c_int64)] * 3 + [c_void_p, c_void_p]),
    "rwb_edge_weights_f32": (c_int32, [c_int32, ctypes.POINTER(c_int64), c_void_p, c_float, c_float,
                                       c_void_p, c_void_p]),
    "rwb_labels_u8": (c_int32, [c_int64, c_void_p, c_void_p, c_void_p]),
    "rwb_downsample_mean_f32": (c_int32, [c_int32, ctypes.POINTER(c_int64), c_void_p, c_void_p, c_void_p]),
    "rwb_downsample_mean_dims_f32": (c_int32, [c_int32, ctypes.POINTER(c_int64), ctypes.c_uint32, c_void_p, c_void_p,
                                               c_void_p]),
    "rwb_chunks_scatter": (c_int32, [c_int32, ctypes.POINTER(c_int64), ctypes.POINTER(c_int64), c_int32, c_void_p,
                                     c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "rwb_const_chunk_table": (c_int32, [c_int32, ctypes.POINTER(c_int64), ctypes.POINTER(c_int64), c_int32, c_void_p,
                                        c_void_p, c_void_p]),
    "rwb_raycast": (c_int32, [c_int32, c_void_p, ctypes.POINTER(c_int64), ctypes.POINTER(ctypes.c_double), c_int64,
                              c_void_p, c_int32, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                              c_int32, c_void_p, c_void_p]),
    "rwb_resample_nn": (c_int32, [c_int32, ctypes.POINTER(c_int64), c_int32, c_int64, c_int32, c_void_p,
                                  ctypes.POINTER(c_int64), ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double), c_void_p, c_void_p]),
    "rwb_chunks_gather": (c_int32, [c_int32, ctypes.POINTER(c_int64), ctypes.POINTER(c_int64), c_int32, c_void_p,
                                    c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "rwb_solve_workspace_bytes": (c_size_t, [c_void_p, c_int64, c_int32]),
    "rwb_solve_level": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
}


class NativeUnavailable(RuntimeError):
    """librwb.so is missing or no sm_100 device is present (no CPU fallback exists)."""


class RWBError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(f"librwb error {code}: {message}")
        self.code = code


class RWBInvalidArgument(RWBError, ValueError):
    """RWB_ERR_INVALID: the library rejected a shape, pointer or parameter."""


class Geometry(ctypes.Structure):
    _fields_ = [("ndim", c_int32), ("reserved", c_int32), ("size", c_int64 * 3),
                ("brick", c_int64 * 3), ("origin", c_int64 * 3)]


class SolveParams(ctypes.Structure):
    _fields_ = [("beta", c_float), ("min_weight", c_float), ("tol", c_float), ("max_iter", c_int32),
                ("check_every", c_int32), ("flags", c_int32)]


class SolveStats(ctypes.Structure):
    _fields_ = [("bricks", c_int64), ("converged", c_int64), ("not_converged", c_int64),
                ("zero_rhs", c_int64), ("iterations_max", c_int64), ("iterations_sum", c_int64),
                ("unknowns", c_int64), ("sweeps", c_int32), ("cg_ms", c_float), ("path", c_int32),
                ("reserved", c_int32), ("unknown_iterations", c_int64)]

    def as_dict(self):
        out = {name: int(getattr(self, name)) for name, _ in self._fields_ if name not in ("cg_ms", "reserved")}
        out["cg_ms"] = float(self.cg_ms)
        return out


_lock = threading.Lock()
_lib = None
_device_checked = False


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load librwb.so and bind every declared symbol (no device required)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.rwb_abi_version() != ABI_VERSION:
            raise NativeUnavailable("librwb ABI version mismatch; rebuild")
        _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    """The library, after checking once that the current device is sm_100."""
    global _device_checked
    handle = load_library()
    if not _device_checked:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the random-walker path runs only on B200 (sm_100a)")
        torch.cuda.init()
        sms, major, minor = c_int32(), c_int32(), c_int32()
        rc = handle.rwb_device_info(ctypes.byref(sms), ctypes.byref(major), ctypes.byref(minor))
        if rc != 0:
            raise NativeUnavailable(handle.rwb_last_error().decode())
        _device_checked = True
    return handle


def check(rc: int):
    if rc != 0:
        msg = load_library().rwb_last_error().decode()
        raise (RWBInvalidArgument if rc == -1 else RWBError)(rc, msg)


def int64_array(values):
    values = [int(v) for v in values]
    return (c_int64 * max(1, len(values)))(*values)
