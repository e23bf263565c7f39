"""Unitary matrix exponentials exp(-iH) on the GPU (reference: expm.py:1-109).

Scaling and squaring with a truncated Taylor series, exactly the reference's
recipe (scale by 2**s until the max-row-sum norm is <= 0.5, order 18, square
s times).  N <= 4 runs one thread per matrix in registers; larger N runs the
Taylor recursion on the FP64 tensor pipe (DMMA complex GEMM with the
``term = term @ a / k; out += term`` epilogue fused).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import NonFinite
from .operators import HermitianOperator

TAYLOR_ORDER = 18
SCALE_TARGET = 0.5
UNITARITY_FRO_TOL = 1e-10
DET_TOL = 1e-8


@dataclass(frozen=True)
class UnitaryPropagator:
    """Dense unitary with optional validation (expm.py:25-47)."""

    entries: np.ndarray

    @property
    def dim(self) -> int:
        return self.entries.shape[0]

    def unitarity_defect(self) -> float:
        """||U U^dag - I||_F (DMMA GEMM with a fused reduction)."""
        t = _lib.require_cuda()
        d_u = _lib.to_device(self.entries)
        out = t.zeros(1, dtype=t.float64, device="cuda")
        _lib.call("qch_unitarity_defect_c128", _lib.dptr(d_u), 1, self.dim, _lib.dptr(out), _lib.stream_ptr())
        return float(out.item())

    def validate(self) -> "UnitaryPropagator":
        d_u = _lib.to_device(self.entries)
        _validate_device(d_u.reshape(1, self.dim, self.dim))
        return self


def _validate_device(d_us) -> None:
    b, n = int(d_us.shape[0]), int(d_us.shape[1])
    bad = ctypes.c_int64(-1)
    st = _lib.load().qch_validate_unitary_batch_c128(_lib.dptr(d_us), b, n, ctypes.byref(bad), _lib.stream_ptr())
    if st != 0:
        raise NonFinite(_lib.last_error())


def _as_dense(h) -> np.ndarray:
    if isinstance(h, HermitianOperator):
        return h.to_dense()
    return np.asarray(h, dtype=np.complex128)


def expm_device(d_h):
    """exp(-i H_b) for a CUDA tensor (batch, n, n); returns a CUDA tensor."""
    t = _lib.require_cuda()
    b, n = int(d_h.shape[0]), int(d_h.shape[1])
    d_u = t.empty_like(d_h)
    work = t.empty((8 * b, n, n), dtype=t.complex128, device="cuda") if n > 4 else None
    bad = ctypes.c_int64(-1)
    st = _lib.load().qch_expm_minus_i_batch_c128(
        _lib.dptr(d_h), b, n, _lib.dptr(d_u), _lib.dptr(work), ctypes.byref(bad), _lib.stream_ptr()
    )
    if st == 6:
        raise NonFinite(f"non-finite entries in batch items [{bad.value}]")
    _lib.check(st)
    return d_u


def expm_unitary(h, *, check: bool = True) -> UnitaryPropagator:
    """exp(-i h) for a dense Hermitian matrix or operator (expm.py:74-86)."""
    mat = _as_dense(h)
    if not np.isfinite(mat).all():
        raise NonFinite("input matrix contains NaN or Inf")
    d_h = _lib.to_device(mat[None])
    d_u = expm_device(d_h)
    if check:
        _validate_device(d_u)
    return UnitaryPropagator(_lib.to_host(d_u[0]))


def expm_batch(hs, *, workers: int | None = None, check: bool = True) -> list[UnitaryPropagator]:
    """Elementwise ``expm_unitary`` over a batch (expm.py:89-109); the whole
    batch is one device call (``workers`` is accepted for API compatibility:
    batch items are parallel on the GPU)."""
    mats = [_as_dense(h) for h in hs]
    bad = [idx for idx, m in enumerate(mats) if not np.isfinite(m).all()]
    if bad:
        raise NonFinite(f"non-finite entries in batch items {bad}")
    if not mats:
        return []
    out: list[UnitaryPropagator] = []
    # group consecutive items of equal dimension into one launch
    start = 0
    while start < len(mats):
        n = mats[start].shape[0]
        stop = start
        while stop < len(mats) and mats[stop].shape[0] == n:
            stop += 1
        d_h = _lib.to_device(np.stack(mats[start:stop]))
        d_u = expm_device(d_h)
        if check:
            _validate_device(d_u)
        host = _lib.to_host(d_u)
        out.extend(UnitaryPropagator(host[k]) for k in range(host.shape[0]))
        start = stop
    return out
