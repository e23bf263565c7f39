"""NPAD: iterative exact block diagonalisation by Givens rotations, on the GPU.

Drop-in for the reference module (npad.py:1-354): same dataclasses, same
functions, same signatures and errors.  Every numerical step runs in
libqcheff's sm_100a kernels:

* ``givens_rotation_matrix``   -> qch_givens_params_c128   (npad.py:101-123)
* ``unitary_transformation``   -> qch_npad_apply_rotations_c128 (npad.py:131-145, 235-241)
* ``eliminate_couplings``      -> ONE launch for all disjoint pairs (npad.py:274-297)
* ``npad_run``                 -> the whole greedy loop on the device (npad.py:300-354)

New API (the parameter-sweep unit of the north star):
* ``npad_run_batch``           -> one persistent block per operator
* ``npad_sweep_transmon``      -> builds the sweep Hamiltonians on the device

Rotation convention (reference docstring, npad.py:1-17): the coupling
``H[j, i] = g e^{i phi}``, ``delta = (H[i,i] - H[j,j]) / 2``,
``r = hypot(delta, g)``, ``cos t = |delta|/r``, ``sin t = sign(delta) g/r``,
``cos(t/2) = sqrt((1 + cos t)/2)``, ``sin(t/2) = sin t / (2 cos(t/2))``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from .errors import IndexOutOfRange, OverlappingPairs, ZeroCoupling
from .operators import HermitianOperator

SPARSE_FILL_DROP = 1e-15  # npad.py:33 (sparse path; operators are densified here)
UNITARY_CHECK_EVERY = 100  # npad.py:36
UNITARY_DRIFT_TOL = 1e-10  # npad.py:37


@dataclass(frozen=True)
class GivensRotation:
    """Two-level unitary on span{|i>, |j>}, i < j (npad.py:40-78).

    Block ``[[c, s e^{-i phase}], [-s e^{i phase}, c]]`` with ``c = cos_half``
    and ``s = sin_half`` (signed).
    """

    i: int
    j: int
    cos_half: float
    sin_half: float
    phase: float
    degenerate: bool = False

    def __post_init__(self):
        if not (0 <= self.i < self.j):
            raise IndexOutOfRange(f"need 0 <= i < j, got ({self.i}, {self.j})")
        residual = abs(self.cos_half**2 + self.sin_half**2 - 1.0)
        if residual > 1e-14:
            raise ValueError(f"rotation parameters not normalized: |c^2+s^2-1| = {residual:.2e}")

    def embedded(self) -> np.ndarray:
        c = self.cos_half
        se = self.sin_half * np.exp(1j * self.phase)
        return np.array([[c, np.conj(se)], [-se, c]], dtype=np.complex128)

    def as_matrix(self, dim: int) -> np.ndarray:
        if self.j >= dim:
            raise IndexOutOfRange(f"rotation indices ({self.i}, {self.j}) exceed dim {dim}")
        u = np.eye(dim, dtype=np.complex128)
        b = self.embedded()
        u[self.i, self.i], u[self.i, self.j] = b[0, 0], b[0, 1]
        u[self.j, self.i], u[self.j, self.j] = b[1, 0], b[1, 1]
        return u


@dataclass
class NPADState:
    """Operator under iteration plus bookkeeping (npad.py:81-98).

    ``accumulated_unitary`` (when tracked) satisfies
    ``current = U @ initial @ U^dag``.
    """

    current: HermitianOperator
    applied: int = 0
    accumulated_unitary: np.ndarray | None = None
    converged: bool = True

    @classmethod
    def from_operator(cls, op: HermitianOperator, *, track_unitary: bool = False) -> "NPADState":
        u = np.eye(op.dim, dtype=np.complex128) if track_unitary else None
        return cls(current=op, accumulated_unitary=u)


# -- device helpers -------------------------------------------------------------

def _params_from_rotations(rots: Sequence[GivensRotation]) -> np.ndarray:
    """Host (c, s) block parameters of given rotations in the kernel layout.
    s = -sin_half * exp(1j*phase) exactly as _block_params (npad.py:126-128)."""
    out = np.zeros((len(rots), 8), dtype=np.float64)
    for k, rot in enumerate(rots):
        s = -rot.sin_half * np.exp(1j * rot.phase)
        out[k] = (rot.cos_half, rot.sin_half, rot.phase, float(rot.degenerate), s.real, s.imag, 0.0, 0.0)
    return out


def _device_params(op: HermitianOperator, pairs: Sequence[tuple[int, int]]):
    """(pairs tensor, params tensor, host params, status) for index pairs."""
    t = _lib.require_cuda()
    dev = op.device_tensor()
    n = len(pairs)
    d_pairs = _lib.to_device(np.asarray(pairs, dtype=np.int64).reshape(n, 2))
    d_params = t.empty((n, 8), dtype=t.float64, device="cuda")
    d_status = t.empty(n, dtype=t.int32, device="cuda")
    _lib.call(
        "qch_givens_params_c128", _lib.dptr(dev), op.dim, _lib.dptr(d_pairs), n, _lib.dptr(d_params),
        _lib.dptr(d_status), _lib.stream_ptr(),
    )
    return d_pairs, d_params, _lib.to_host(d_params), _lib.to_host(d_status)


def _check_pair(op: HermitianOperator, i: int, j: int) -> None:
    if not (0 <= i < j < op.dim):
        raise IndexOutOfRange(f"need 0 <= i < j < {op.dim}, got ({i}, {j})")


def _rotation_from_row(i: int, j: int, row: np.ndarray) -> GivensRotation:
    return GivensRotation(int(i), int(j), float(row[0]), float(row[1]), float(row[2]), degenerate=bool(row[3] != 0.0))


def _nonherm(dev) -> int:
    t = _lib.torch()
    flag = t.zeros(1, dtype=t.int32, device="cuda")
    _lib.call("qch_hermitian_exact_c128", _lib.dptr(dev), int(dev.shape[0]), _lib.dptr(flag), _lib.stream_ptr())
    return int(flag.item())


def _apply(op: HermitianOperator, d_pairs, d_params, n_pairs: int, u_host):
    """Copy op's matrix on the device, apply the rotations; returns the new
    operator and the updated accumulated unitary (host) if given."""
    dev = op.device_tensor()
    out = dev.clone()
    herm = 0 if _nonherm(out) else 1
    d_u = _lib.to_device(u_host) if u_host is not None else None
    _lib.call(
        "qch_npad_apply_rotations_c128", _lib.dptr(out), op.dim, _lib.dptr(d_pairs), _lib.dptr(d_params), n_pairs,
        herm, _lib.dptr(d_u), _lib.stream_ptr(),
    )
    new_u = _lib.to_host(d_u) if d_u is not None else None
    return HermitianOperator._from_device(out), new_u, d_u


def _audit(d_u, applied: int, dim: int) -> None:
    """UnitarityDrift audit of npad.py:254-259 on the device."""
    from .errors import UnitarityDrift

    t = _lib.torch()
    out = t.zeros(1, dtype=t.float64, device="cuda")
    _lib.call("qch_unitarity_defect_c128", _lib.dptr(d_u), 1, dim, _lib.dptr(out), _lib.stream_ptr())
    drift = float(out.item())
    if drift > UNITARY_DRIFT_TOL * dim:
        raise UnitarityDrift(f"accumulated unitary drift {drift:.3e} after {applied} rotations")


# -- sparse CSR path (npad.py:148-232) -------------------------------------------------

def _is_sparse(op: HermitianOperator) -> bool:
    return op.layout == "sparse"


def _sparse_rotation(op: HermitianOperator, i: int, j: int) -> GivensRotation:
    """givens_rotation_matrix (npad.py:101-123) on a sparse operator: the three
    entries come from the device CSR, the scalars are formed exactly as the
    reference forms them (Python / numpy scalar math)."""
    import math

    t = _lib.require_cuda()
    ip, ix, dv = op.device_csr()
    out = t.empty(3, dtype=t.complex128, device="cuda")
    _lib.call("qch_npad_sparse_entries_c128", _lib.dptr(ip), _lib.dptr(ix), _lib.dptr(dv), op.dim, i, j,
              _lib.dptr(out), _lib.stream_ptr())
    v, hii, hjj = (complex(z) for z in _lib.to_host(out))
    if v == 0:
        raise ZeroCoupling(f"entry ({j}, {i}) is zero; nothing to eliminate")
    g = abs(v)
    phi = float(np.angle(v))
    delta = (hii.real - hjj.real) / 2.0
    r = math.hypot(delta, g)
    sgn = 1.0 if delta >= 0.0 else -1.0
    cos_t = abs(delta) / r
    sin_t = sgn * g / r
    cos_half = math.sqrt((1.0 + cos_t) / 2.0)
    sin_half = sin_t / (2.0 * cos_half)
    return GivensRotation(i, j, cos_half, sin_half, phi, degenerate=(delta == 0.0))


def _sparse_transform(op: HermitianOperator, rot: GivensRotation) -> HermitianOperator:
    """U H U^dag on the device CSR (qch_npad_sparse_rotate_c128): a new sparse
    operator, bit-identical to the reference's _conjugate_sparse."""
    t = _lib.require_cuda()
    ip, ix, dv = op.device_csr()
    nnz = int(dv.numel())
    ends = _lib.to_host(ip[[rot.i, rot.i + 1, rot.j, rot.j + 1]])
    cap = nnz + 4 * int((ends[1] - ends[0]) + (ends[3] - ends[2])) + 8
    out_ip = t.empty(op.dim + 1, dtype=t.int64, device="cuda")
    out_ix = t.empty(cap, dtype=t.int32, device="cuda")
    out_dv = t.empty(cap, dtype=t.complex128, device="cuda")
    s = -rot.sin_half * np.exp(1j * rot.phase)  # _block_params (npad.py:126-128)
    nnz_out = ctypes.c_int64(0)
    _lib.check(_lib.load().qch_npad_sparse_rotate_c128(
        _lib.dptr(ip), _lib.dptr(ix), _lib.dptr(dv), op.dim, nnz, rot.i, rot.j, float(rot.cos_half), float(s.real),
        float(s.imag), float(op.max_abs()), _lib.dptr(out_ip), _lib.dptr(out_ix), _lib.dptr(out_dv), cap,
        ctypes.byref(nnz_out), _lib.stream_ptr()))
    k = int(nnz_out.value)
    return HermitianOperator._from_device_csr(out_ip, out_ix[:k], out_dv[:k], op.dim)


# -- reference API -----------------------------------------------------------------

def givens_rotation_matrix(op: HermitianOperator, i: int, j: int) -> GivensRotation:
    """Rotation zeroing the (i, j) coupling of ``op`` (npad.py:101-123).

    ZeroCoupling when H[j, i] == 0; a degenerate pair (delta == 0) is flagged.
    """
    _check_pair(op, i, j)
    if _is_sparse(op):
        return _sparse_rotation(op, i, j)
    _, _, params, status = _device_params(op, [(i, j)])
    if status[0] != 0:
        raise ZeroCoupling(f"entry ({j}, {i}) is zero; nothing to eliminate")
    return _rotation_from_row(i, j, params[0])


def unitary_transformation(op: HermitianOperator, rot: GivensRotation) -> HermitianOperator:
    """U H U^dag for one rotation; only rows/columns i, j change (npad.py:235-241)."""
    if rot.j >= op.dim:
        raise IndexOutOfRange(f"rotation indices ({rot.i}, {rot.j}) exceed dim {op.dim}")
    if _is_sparse(op):
        return _sparse_transform(op, rot)
    d_pairs = _lib.to_device(np.array([[rot.i, rot.j]], dtype=np.int64))
    d_params = _lib.to_device(_params_from_rotations([rot]))
    new_op, _, _ = _apply(op, d_pairs, d_params, 1, None)
    return new_op


def eliminate_coupling(state: NPADState, i: int, j: int) -> NPADState:
    """Zero one coupling (npad.py:262-271)."""
    return eliminate_couplings(state, [(i, j)])


def eliminate_couplings(state: NPADState, pairs: Sequence[tuple[int, int]]) -> NPADState:
    """Zero several index-disjoint couplings with rotations all built from the
    same input operator, applied in list order — one fused launch
    (npad.py:274-297)."""
    pairs = [(int(a), int(b)) for a, b in pairs]
    if not pairs:
        return state
    flat = [k for pair in pairs for k in pair]
    if len(set(flat)) != len(flat):
        raise OverlappingPairs(f"index pairs share an index: {pairs}")
    op = state.current
    for i, j in pairs:
        _check_pair(op, i, j)
    u_host = state.accumulated_unitary
    # the reference audits U after every rotation that brings the count to a
    # multiple of UNITARY_CHECK_EVERY (npad.py:290-296): apply the pairs in
    # segments ending at those points, auditing after each
    cuts = [k + 1 for k in range(len(pairs)) if (state.applied + k + 1) % UNITARY_CHECK_EVERY == 0]
    bounds = sorted(set([0] + (cuts if u_host is not None else []) + [len(pairs)]))
    if _is_sparse(op):
        # the reference's sparse branch: every rotation built from the input
        # operator, applied in list order (npad.py:287-296); U (if tracked)
        # is a dense device matrix updated by rows, the operator stays a CSR
        rots = [_sparse_rotation(op, i, j) for i, j in pairs]
        d_u = _lib.to_device(u_host) if u_host is not None else None
        cur = op
        for a, b in zip(bounds, bounds[1:]):
            for rot in rots[a:b]:
                cur = _sparse_transform(cur, rot)
            if d_u is not None:
                d_pairs = _lib.to_device(np.array([[r.i, r.j] for r in rots[a:b]], dtype=np.int64))
                d_params = _lib.to_device(_params_from_rotations(rots[a:b]))
                _lib.call("qch_npad_apply_rotations_c128", None, op.dim, _lib.dptr(d_pairs), _lib.dptr(d_params),
                          b - a, 0, _lib.dptr(d_u), _lib.stream_ptr())
                if (state.applied + b) % UNITARY_CHECK_EVERY == 0:
                    _audit(d_u, state.applied + b, op.dim)
        return replace(state, current=cur, applied=state.applied + len(pairs),
                       accumulated_unitary=_lib.to_host(d_u) if d_u is not None else None)
    d_pairs, d_params, _, status = _device_params(op, pairs)
    bad = np.flatnonzero(status)
    if bad.size:
        i, j = pairs[int(bad[0])]
        raise ZeroCoupling(f"entry ({j}, {i}) is zero; nothing to eliminate")
    cur = op
    for a, b in zip(bounds, bounds[1:]):
        cur, u_host, d_u = _apply(cur, d_pairs[a:b].contiguous(), d_params[a:b].contiguous(), b - a, u_host)
        if d_u is not None and (state.applied + b) % UNITARY_CHECK_EVERY == 0:
            _audit(d_u, state.applied + b, op.dim)
    return replace(state, current=cur, applied=state.applied + len(pairs), accumulated_unitary=u_host)


def _target_tensor(target, dim: int):
    if target is None:
        return None, 0
    tset = sorted(frozenset(int(k) for k in target))
    if tset and (max(tset) >= dim or min(tset) < 0):
        raise IndexOutOfRange("target indices exceed operator dimension")
    arr = np.asarray(tset, dtype=np.int32)
    if arr.size == 0:
        arr = np.zeros(1, dtype=np.int32)  # valid pointer, n_target = 0
        return _lib.to_device(arr), 0
    return _lib.to_device(arr), len(tset)


def _npad_run_sparse(op, target, tol, max_iter, pivot_cap):
    """The reference's greedy loop (npad.py:320-354) on a sparse operator: each
    step selects the largest relevant coupling of the device CSR
    (qch_npad_sparse_select_c128) and applies the sparse rotation — the
    operator stays sparse and fill-in is dropped exactly as the reference's
    _conjugate_sparse drops it."""
    t = _lib.require_cuda()
    d_target, n_target = _target_tensor(target, op.dim)
    mask = None
    if d_target is not None:
        mask = t.zeros(op.dim, dtype=t.uint8, device="cuda")
        if n_target:
            mask[d_target[:n_target].long()] = 1
    threshold = tol * op.max_abs()
    ek = 1 if (op.max_abs() > 1e100 or (0.0 < threshold < 1e-140)) else 0
    state = NPADState.from_operator(op)
    cur = op
    pivots = []
    out = (ctypes.c_double * 3)()
    applied = 0
    converged = False
    while True:
        ip, ix, dv = cur.device_csr()
        _lib.call("qch_npad_sparse_select_c128", _lib.dptr(ip), _lib.dptr(ix), _lib.dptr(dv), cur.dim,
                  _lib.dptr(mask), ek, out, _lib.stream_ptr())
        i, j, mag = int(out[0]), int(out[1]), float(out[2])
        if i < 0 or mag < threshold:
            converged = True
            break
        if applied >= max_iter:
            break
        if len(pivots) < pivot_cap:
            pivots.append((i, j))
        rot = _sparse_rotation(cur, i, j)
        cur = _sparse_transform(cur, rot)
        applied += 1
    state = NPADState(current=cur, applied=applied, accumulated_unitary=None, converged=converged)
    piv = np.asarray(pivots, dtype=np.int32).reshape(-1, 2)
    return state, piv


def _npad_run_device(op, target, tol, max_iter, track_unitary, pivot_cap=0):
    if tol <= 0:
        raise ValueError("tol must be positive")
    if max_iter is None:
        max_iter = 20 * op.dim * op.dim
    if op.layout == "sparse" and not track_unitary:
        if target is not None and any(int(k) >= op.dim for k in target):
            raise IndexOutOfRange("target indices exceed operator dimension")
        return _npad_run_sparse(op, target, tol, max_iter, pivot_cap)
    t = _lib.require_cuda()
    d_target, n_target = _target_tensor(target, op.dim)
    threshold = tol * op.max_abs()
    work = op.device_tensor().clone()
    d_u = t.eye(op.dim, dtype=t.complex128, device="cuda") if track_unitary else None
    d_piv = t.full((max(pivot_cap, 1), 2), -1, dtype=t.int32, device="cuda") if pivot_cap > 0 else None
    applied = ctypes.c_int64(0)
    conv = ctypes.c_int(0)
    _lib.call(
        "qch_npad_run_dense_c128", _lib.dptr(work), op.dim, _lib.dptr(d_target), n_target, float(threshold),
        int(max_iter), _lib.dptr(d_u), _lib.dptr(d_piv), int(pivot_cap), ctypes.byref(applied), ctypes.byref(conv),
        _lib.stream_ptr(),
    )
    state = NPADState(
        current=HermitianOperator._from_device(work),
        applied=int(applied.value),
        accumulated_unitary=_lib.to_host(d_u) if d_u is not None else None,
        converged=bool(conv.value),
    )
    pivots = None
    if d_piv is not None:
        pivots = _lib.to_host(d_piv)[: min(state.applied, pivot_cap)]
    return state, pivots


def npad_run(
    op: HermitianOperator,
    target: Iterable[int] | None = None,
    *,
    tol: float,
    max_iter: int | None = None,
    track_unitary: bool = False,
) -> NPADState:
    """Eliminate the largest remaining coupling until convergence (npad.py:320-354).

    ``target=None`` drives toward a full diagonal; a set of indices decouples
    that subspace (only couplings with exactly one endpoint inside count).
    Converged when every relevant magnitude is below ``tol * max|op|``;
    reaching ``max_iter`` (default ``20 * dim**2``) returns
    ``converged=False``.  The entire greedy chain runs on the device.
    """
    state, _ = _npad_run_device(op, target, tol, max_iter, track_unitary)
    return state


def npad_run_logged(op, target=None, *, tol, max_iter=None, track_unitary=False, pivot_cap=None):
    """``npad_run`` plus the (i, j) pivot sequence (int32 array, one row per
    rotation) — the parity harness's view of the greedy order."""
    if pivot_cap is None:
        pivot_cap = max_iter if max_iter is not None else 20 * op.dim * op.dim
    return _npad_run_device(op, target, tol, max_iter, track_unitary, pivot_cap=int(pivot_cap))


# -- new API: batched sweeps ----------------------------------------------------------

@dataclass
class BatchResult:
    """Result of a batched npad_run: device-resident final operators, rotation
    counts and convergence flags.  ``parts`` holds (first item, (b, n, n)
    CUDA tensor) per device (one part unless ``devices`` spread the batch)."""

    parts: list
    applied: np.ndarray
    converged: np.ndarray

    @property
    def matrices(self):
        """(batch, n, n) CUDA tensor of the final operators (single-device
        results; multi-device results are in ``parts``)."""
        if len(self.parts) != 1:
            raise ValueError("result spans several devices: use .parts or .operator(b)")
        return self.parts[0][1]

    def _locate(self, b: int):
        for start, mats in reversed(self.parts):
            if b >= start:
                return mats, b - start
        raise IndexError(b)

    def operator(self, b: int) -> HermitianOperator:
        mats, k = self._locate(b)
        return HermitianOperator._from_device(mats[k])

    def diagonals(self) -> np.ndarray:
        # one part (one device): the page-locked array to_host filled is the
        # result — concatenating would copy it into fresh pageable pages
        arrs = [_lib.to_host(m.diagonal(dim1=1, dim2=2).real.contiguous()) for _, m in self.parts]
        return arrs[0] if len(arrs) == 1 else np.concatenate(arrs)


def max_abs_batch(mats):
    """Per-item max |H| of a (b, n, n) device batch, ONE launch
    (qch_max_abs_batch_c128, numpy |z| as operators.py:92-99)."""
    t = _lib.require_cuda()
    b = int(mats.shape[0])
    out = t.empty(b, dtype=t.float64, device=mats.device)
    _lib.call("qch_max_abs_batch_c128", _lib.dptr(mats), b, int(mats[0].numel()), _lib.dptr(out), _lib.stream_ptr())
    return out


def _run_batch_inplace(mats, target, tol, max_iter, max_abs_dev=None, sync=True):
    t = _lib.require_cuda()
    b, n = int(mats.shape[0]), int(mats.shape[1])
    if tol <= 0:
        raise ValueError("tol must be positive")
    if max_iter is None:
        max_iter = 20 * n * n
    d_target, n_target = _target_tensor(target, n)
    if max_abs_dev is None:
        max_abs_dev = max_abs_batch(mats)
    thr = max_abs_dev * float(tol)
    applied = t.empty(b, dtype=t.int64, device=mats.device)
    conv = t.empty(b, dtype=t.int32, device=mats.device)
    _lib.call(
        "qch_npad_run_batch_c128", _lib.dptr(mats), b, n, _lib.dptr(d_target), n_target, _lib.dptr(thr),
        int(max_iter), _lib.dptr(applied), _lib.dptr(conv), _lib.stream_ptr(),
    )
    return applied, conv


def _batch_on_current_device(ops, target, tol, max_iter):
    """One device: bitwise-Hermitian operators go through the batched
    many-chain driver; any others (Hermitian only to rounding, which the
    batched lazy-column driver cannot take) through npad_run one by one —
    the same per-operator results either way."""
    t = _lib.require_cuda()
    mats = t.stack([op.device_tensor().to(t.cuda.current_device()) for op in ops]).contiguous()
    b = len(ops)
    herm = [not _nonherm(mats[k]) for k in range(b)]
    applied = np.zeros(b, dtype=np.int64)
    conv = np.zeros(b, dtype=bool)
    idx = [k for k in range(b) if herm[k]]
    if idx:
        sub = mats[idx].contiguous() if len(idx) < b else mats
        max_abs = t.tensor([ops[k].max_abs() for k in idx], dtype=t.float64, device=mats.device)
        ap, cv = _run_batch_inplace(sub, target, tol, max_iter, max_abs)
        applied[idx] = _lib.to_host(ap)
        conv[idx] = _lib.to_host(cv).astype(bool)
        if len(idx) < b:
            mats[idx] = sub
    for k in range(b):
        if not herm[k]:
            st = npad_run(HermitianOperator._from_device(mats[k].clone()), target, tol=tol, max_iter=max_iter)
            mats[k].copy_(st.current.device_tensor())
            applied[k], conv[k] = st.applied, st.converged
    return mats, applied, conv


def npad_run_batch(ops: Sequence[HermitianOperator], target=None, *, tol: float, max_iter: int | None = None,
                   devices: Sequence[int] | None = None) -> BatchResult:
    """``npad_run`` over independent operators of one dimension (new API;
    per-point results equal ``npad_run`` on each operator): one warp-resident
    chain per operator.  ``devices``: CUDA device ordinals to spread the batch
    over (contiguous blocks, one host thread per device, no communication);
    default the current device."""
    _lib.require_cuda()
    ops = list(ops)
    if not ops:
        raise ValueError("need at least one operator")
    if tol <= 0:
        raise ValueError("tol must be positive")
    devs = list(devices) if devices else [None]
    if len(devs) == 1:
        if devs[0] is None:
            mats, ap, cv = _batch_on_current_device(ops, target, tol, max_iter)
        else:
            with _lib.torch().cuda.device(int(devs[0])):
                mats, ap, cv = _batch_on_current_device(ops, target, tol, max_iter)
        return BatchResult([(0, mats)], ap, cv)
    import threading

    from .sharding import shard_bounds

    t = _lib.torch()
    res, errs = {}, []

    def work(r, dev):
        try:
            a, b = shard_bounds(len(ops), len(devs), r)
            if a == b:
                return
            with t.cuda.device(int(dev)):
                mats, ap, cv = _batch_on_current_device(ops[a:b], target, tol, max_iter)
                t.cuda.current_stream().synchronize()
            res[r] = (a, mats, ap, cv)
        except BaseException as e:  # re-raised on the calling thread
            errs.append(e)

    th = [threading.Thread(target=work, args=(r, d)) for r, d in enumerate(devs)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    if errs:
        raise errs[0]
    parts = [res[r] for r in sorted(res)]
    return BatchResult([(a, m) for a, m, _, _ in parts], np.concatenate([p[2] for p in parts]),
                       np.concatenate([p[3] for p in parts]))


def build_transmon_resonator_batch(params: np.ndarray, n_q: int, n_r: int, *, with_max_abs: bool = False):
    """Device-built transmon (x) resonator Hamiltonians, one per row of
    ``params`` = (omega_q, alpha, omega_r, g).  Same matrix as
    models.transmon_resonator_hamiltonian.  ``with_max_abs``: also return
    each operator's max |H| (formed by the builder, no extra pass)."""
    t = _lib.require_cuda()
    params = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 4)
    b = params.shape[0]
    n = n_q * n_r
    mats = t.empty((b, n, n), dtype=t.complex128, device="cuda")
    mx = t.empty(b, dtype=t.float64, device="cuda") if with_max_abs else None
    d_prm = _lib.to_device(params)
    _lib.call("qch_build_transmon_resonator_c128", _lib.dptr(mats), b, n_q, n_r, _lib.dptr(d_prm), _lib.dptr(mx),
              _lib.stream_ptr())
    return (mats, mx) if with_max_abs else mats


def npad_sweep_transmon(params: np.ndarray, n_q: int, n_r: int, target=None, *, tol: float,
                        max_iter: int | None = None) -> BatchResult:
    """Parameter sweep of config 4: build every (omega_q, alpha, omega_r, g)
    point on the device and run the batched greedy NPAD (new API)."""
    mats, mx = build_transmon_resonator_batch(params, n_q, n_r, with_max_abs=True)
    applied, conv = _run_batch_inplace(mats, target, tol, max_iter, mx)
    return BatchResult([(0, mats)], _lib.to_host(applied), _lib.to_host(conv).astype(bool))
