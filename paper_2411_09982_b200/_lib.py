"""ctypes binding of libqcheff.so (include/qcheff.h) and device plumbing.

PyTorch is used only for device memory and the current CUDA stream; every
numerical operation of the hot paths runs in the hand-written kernels of the
library.  There is deliberately no CPU fallback: on a machine without a CUDA
device, or without the built library, every hot-path call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from . import errors

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libqcheff.so"
_lock = threading.Lock()
_lib = None

c_void_p = ctypes.c_void_p
c_int64 = ctypes.c_int64
c_int = ctypes.c_int
c_double = ctypes.c_double
P_int64 = ctypes.POINTER(ctypes.c_int64)
P_int = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes); mirrors include/qcheff.h
PROTOTYPES = {
    "qch_version": (c_int, []),
    "qch_last_error": (ctypes.c_size_t, [ctypes.c_char_p, ctypes.c_size_t]),
    "qch_launch_count": (c_int64, []),
    "qch_max_abs_c128": (c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    "qch_max_abs_batch_c128": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "qch_hermitian_exact_c128": (c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    "qch_hermitian_defect_c128": (c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    "qch_givens_params_c128": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "qch_npad_apply_rotations_c128": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "qch_npad_run_dense_c128": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_double, c_int64, c_void_p, c_void_p, c_int64, P_int64, P_int, c_void_p],
    ),
    "qch_npad_run_batch_c128": (
        c_int,
        [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p],
    ),
    "qch_build_transmon_resonator_c128": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "qch_magnus_coefficients": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_double, c_int, c_void_p, c_void_p, c_void_p]),
    "qch_magnus_commutators_c128": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "qch_magnus_assemble_c128": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_int64, c_int64, c_double, c_int, c_void_p, c_void_p],
    ),
    "qch_expm_minus_i_batch_c128": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, P_int64, c_void_p]),
    "qch_expm_norm_c128": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "qch_validate_unitary_batch_c128": (c_int, [c_void_p, c_int64, c_int64, P_int64, c_void_p]),
    "qch_unitarity_defect_c128": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "qch_magnus_evolve_c128": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_double, c_double, c_int64, c_int,
         c_void_p, c_void_p, c_void_p, c_int, P_int64, c_void_p],
    ),
    "qch_magnus_shard_workspace_bytes": (c_int64, [c_int64, c_int64]),
    "qch_magnus_shard_prepare_c128": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_double, c_double, c_int64, c_int, c_int,
         c_void_p, c_void_p, c_void_p],
    ),
    "qch_magnus_apply_prefix_c128": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "qch_magnus_shard_finish_c128": (c_int, [c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int, P_int64, c_void_p]),
    "qch_magnus_shard_finish_async_c128": (
        c_int, [c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "qch_npad_sparse_rotate_c128": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_double, c_double, c_double, c_double,
         c_void_p, c_void_p, c_void_p, c_int64, P_int64, c_void_p],
    ),
    "qch_npad_sparse_select_c128": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int, c_void_p,
                                            c_void_p]),
    "qch_build_ladder_csr_c128": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "qch_build_spin_chain_drift_c128": (c_int, [c_int64, c_double, c_double, c_double, c_void_p, c_void_p, c_void_p,
                                                P_int64, c_void_p]),
    "qch_build_global_xy_c128": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p]),
    "qch_npad_sparse_entries_c128": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p,
                                             c_void_p]),
    "qch_peak_kernel": (c_int, [c_int, c_int, c_int, c_void_p, ctypes.POINTER(c_double), c_void_p]),
    "qch_profile_enable": (None, [c_int]),
    "qch_profile_read": (c_int, [c_void_p, c_void_p, ctypes.c_char_p, c_int64, c_int, c_int]),
    "qch_magnus_evolve_async_c128": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_double, c_double, c_int64, c_int,
         c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p],
    ),
    "qch_magnus_plan_workspace_bytes": (c_int64, [c_int64, c_int64]),
    "qch_rk4_evolve_c128": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_double,
                                    c_double, c_int64, c_void_p, c_void_p, c_void_p]),
    "qch_magnus_plan_workspace_init": (c_int, [c_void_p, c_int64, c_int64, c_void_p]),
    "qch_magnus_evolve_plan_c128": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_double, c_double, c_int64, c_int,
         c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p],
    ),
    "qch_magnus_evolve_host_c128": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_double, c_double, c_int64, c_int, c_void_p,
         c_void_p, c_int, P_int64, c_void_p, c_void_p],
    ),
    "qch_zgemm_batched": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p],
    ),
    "qch_magnus_propagators_c128": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_double, c_double, c_int64, c_int,
         c_int, c_void_p, P_int64, c_void_p],
    ),
    "qch_magnus_chain_c128": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, P_int64, c_void_p]),
    "qch_zgemm_herm_batched": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p]),
    "qch_zgemm_real_products": (c_int, []),
    "qch_dmma_flops": (c_double, []),
    "qch_set_herm_gemm": (c_int, [c_int]),
    "qch_int8_ops": (c_double, []),
    "qch_int8_fp64_equiv_flops": (c_double, []),
    "qch_i8gemm_test": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    "qch_oz_real_test": (
        c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p]),
}

QCH_OK = 0
STATUS_TO_ERROR = {
    1: ValueError,
    2: errors.IndexOutOfRange,
    3: errors.ZeroCoupling,
    4: errors.OverlappingPairs,
    5: errors.UnitarityDrift,
    6: errors.NonFinite,
    7: errors.GridMismatch,
    8: errors.DimensionMismatch,
    9: errors.NormDrift,
    10: errors.HermiticityViolation,
    11: NotImplementedError,
    12: RuntimeError,
}


def lib_path() -> Path:
    return _LIB_PATH


def load(build_if_missing: bool = True):
    """Load (building in-tree first if needed) and type the shared library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_missing and os.environ.get("QCH_AUTOBUILD", "1") == "1":
            from . import _build

            if _build.stale():
                _build.build()
        if not _LIB_PATH.exists():
            raise RuntimeError(f"{_LIB_PATH} is missing; run __graft_entry__.build()")
        lib = ctypes.CDLL(str(_LIB_PATH))
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    lib = load()
    buf = ctypes.create_string_buffer(1024)
    lib.qch_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(status: int) -> None:
    if status == QCH_OK:
        return
    exc = STATUS_TO_ERROR.get(status, RuntimeError)
    raise exc(last_error())


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def launch_count() -> int:
    return int(load().qch_launch_count())


def profile_enable(on: bool) -> None:
    load().qch_profile_enable(1 if on else 0)


def profile_read(reset: bool = True) -> dict:
    """{kernel name: (total_ms, launches)} recorded since the last reset."""
    lib = load()
    cap = 64
    tot = (c_double * cap)()
    cnt = (c_int64 * cap)()
    buf = ctypes.create_string_buffer(8192)
    k = lib.qch_profile_read(ctypes.cast(tot, c_void_p), ctypes.cast(cnt, c_void_p), buf, len(buf), cap,
                             1 if reset else 0)
    names = buf.raw.split(b"\0")
    return {names[i].decode(): (float(tot[i]), int(cnt[i])) for i in range(min(k, cap))}


# -- device plumbing (torch owns memory and streams) ---------------------------

def torch():
    import torch as _t

    return _t


_cuda_ok = False


def require_cuda():
    global _cuda_ok
    t = torch()
    if _cuda_ok:
        return t
    if not t.cuda.is_available():
        raise RuntimeError(
            "paper_2411_09982_b200 needs a CUDA device: the hot paths run only in libqcheff's sm_100a kernels "
            "(there is no CPU fallback)"
        )
    load()
    _cuda_ok = True
    return t


def cuda_available() -> bool:
    """True when a CUDA device and the library are usable (validation
    helpers move large scans to the device; the hot paths require it)."""
    try:
        require_cuda()
        return True
    except RuntimeError:
        return False


def stream_ptr():
    t = torch()
    return c_void_p(t.cuda.current_stream().cuda_stream)


def dptr(tensor) -> c_void_p:
    if tensor is None:
        return c_void_p(None)
    return c_void_p(tensor.data_ptr())


def to_device(array, dtype=None):
    """Host array -> contiguous CUDA tensor (complex128 / float64 / int)."""
    t = require_cuda()
    if isinstance(array, t.Tensor):
        out = array
        if not out.is_cuda:
            out = out.cuda()
        if dtype is not None and out.dtype != dtype:
            out = out.to(dtype)
        return out.contiguous()
    arr = np.ascontiguousarray(array)
    out = t.from_numpy(arr)
    if dtype is not None:
        out = out.to(dtype)
    return out.cuda(non_blocking=False).contiguous()


PINNED_MIN_BYTES = 1 << 16


def host_empty(shape, dtype=np.complex128) -> np.ndarray:
    """Uninitialised numpy array in page-locked host memory (torch's caching
    host allocator: freed blocks are reused, so steady-state calls do not
    cudaHostAlloc).  DMA targets for the host-buffer C-ABI calls."""
    t = torch()
    tdt = {np.dtype(np.complex128): t.complex128, np.dtype(np.float64): t.float64}[np.dtype(dtype)]
    return t.empty(tuple(shape), dtype=tdt, pin_memory=True).numpy()


def to_host(tensor) -> np.ndarray:
    """Device tensor -> numpy.  Large results land in pinned memory (full-speed
    DMA, no pageable staging copy)."""
    tensor = tensor.detach()
    if tensor.is_cuda and tensor.numel() * tensor.element_size() >= PINNED_MIN_BYTES:
        t = torch()
        out = t.empty(tensor.shape, dtype=tensor.dtype, pin_memory=True)
        out.copy_(tensor, non_blocking=True)
        t.cuda.current_stream().synchronize()
        return out.numpy()
    return tensor.cpu().numpy()


def ptr(array: np.ndarray) -> c_void_p:
    """Host address of a C-contiguous numpy array."""
    return c_void_p(array.ctypes.data)
