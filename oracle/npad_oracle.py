"""NPAD restatement (reference npad.py / operators.py), numpy, in place.

Two drivers with identical results:
* ``run_full_scan``   — literal restatement: every step rescans the strict
  lower triangle like _largest_relevant (npad.py:300-317).
* ``run_incremental`` — per-row maxima maintained across rotations (the
  algorithm of the GPU kernel); bit-identical pivots and
  matrix, O(N) per rotation, so it can check N = 4096.
"""
from __future__ import annotations

import math

import numpy as np


def max_abs(h: np.ndarray) -> float:
    """operators.py:98."""
    return float(np.max(np.abs(h))) if h.size else 0.0


def pick_full_scan(h: np.ndarray, mask: np.ndarray | None):
    """Largest relevant coupling (npad.py:300-317 over operators.py:133-139):
    returns (i, j, mag) with the pivot at H[j, i], j > i, or None."""
    rows, cols = np.nonzero(np.tril(h, k=-1))
    vals = h[rows, cols]
    if mask is not None and rows.size:
        sel = mask[rows] != mask[cols]
        rows, cols, vals = rows[sel], cols[sel], vals[sel]
    if rows.size == 0:
        return None
    mags = np.abs(vals)
    best = np.lexsort((rows, cols, -mags))[0]
    if mags[best] == 0.0:
        return None
    return int(cols[best]), int(rows[best]), float(mags[best])


def rotation_scalars(h: np.ndarray, i: int, j: int):
    """givens_rotation_matrix (npad.py:101-123): (cos_half, sin_half, phase,
    degenerate).  Caller guarantees H[j, i] != 0."""
    v = complex(h[j, i])
    g = abs(v)
    phase = float(np.angle(v))
    delta = (complex(h[i, i]).real - complex(h[j, j]).real) / 2.0
    radius = math.hypot(delta, g)
    sign = 1.0 if delta >= 0.0 else -1.0
    cos_t = abs(delta) / radius
    sin_t = sign * g / radius
    cos_half = math.sqrt((1.0 + cos_t) / 2.0)
    return cos_half, sin_t / (2.0 * cos_half), phase, delta == 0.0


def block_s(sin_half: float, phase: float):
    """s of the block [[c, -conj(s)], [s, c]] (npad.py:126-128)."""
    return -sin_half * np.exp(1j * phase)


def rotate(h: np.ndarray, i: int, j: int, c: float, s) -> None:
    """_conjugate_dense (npad.py:131-145) without the defensive copy."""
    row_i, row_j = h[i, :].copy(), h[j, :].copy()
    h[i, :] = c * row_i - np.conj(s) * row_j
    h[j, :] = s * row_i + c * row_j
    col_i, col_j = h[:, i].copy(), h[:, j].copy()
    h[:, i] = c * col_i - s * col_j
    h[:, j] = np.conj(s) * col_i + c * col_j
    h[i, i] = h[i, i].real
    h[j, j] = h[j, j].real
    h[j, i] = np.conj(h[i, j])


def rotate_unitary(u: np.ndarray, i: int, j: int, c: float, s) -> None:
    """_apply_left (npad.py:244-251) in place."""
    row_i, row_j = u[i, :].copy(), u[j, :].copy()
    u[i, :] = c * row_i - np.conj(s) * row_j
    u[j, :] = s * row_i + c * row_j


def unitary_drift(u: np.ndarray) -> float:
    """npad.py:257."""
    return float(np.linalg.norm(u @ u.conj().T - np.eye(u.shape[0])))


def _mask(n: int, target):
    if target is None:
        return None
    m = np.zeros(n, dtype=bool)
    m[list(target)] = True
    return m


def run_full_scan(h0: np.ndarray, target=None, *, tol: float, max_iter=None, track_unitary=False):
    """npad_run (npad.py:320-354).  Returns dict(h, applied, converged,
    pivots (applied, 2), u)."""
    h = np.array(h0, dtype=np.complex128, copy=True)
    n = h.shape[0]
    if max_iter is None:
        max_iter = 20 * n * n
    threshold = tol * max_abs(h)
    mask = _mask(n, target)
    u = np.eye(n, dtype=np.complex128) if track_unitary else None
    pivots = []
    while True:
        pick = pick_full_scan(h, mask)
        if pick is None or pick[2] < threshold:
            converged = True
            break
        if len(pivots) >= max_iter:
            converged = False
            break
        i, j, _ = pick
        c, sh, ph, _ = rotation_scalars(h, i, j)
        s = block_s(sh, ph)
        rotate(h, i, j, c, s)
        if u is not None:
            rotate_unitary(u, i, j, c, s)
        pivots.append((i, j))
    return dict(h=h, applied=len(pivots), converged=converged, pivots=np.asarray(pivots, dtype=np.int64).reshape(-1, 2),
                u=u)


class _RowMax:
    """Per-row (max |H[r, c]|, argmin-col among ties) over relevant c < r."""

    def __init__(self, h: np.ndarray, mask):
        self.h = h
        self.mask = mask
        n = h.shape[0]
        self.val = np.full(n, -1.0)
        self.col = np.full(n, -1, dtype=np.int64)
        for r in range(n):
            self.rescan(r)

    def rescan(self, r: int) -> None:
        if r == 0:
            self.val[r], self.col[r] = -1.0, -1
            return
        mags = np.abs(self.h[r, :r])
        if self.mask is not None:
            mags = np.where(self.mask[:r] != self.mask[r], mags, -1.0)
        k = int(np.argmax(mags))
        if mags[k] < 0.0:
            self.val[r], self.col[r] = -1.0, -1
        else:
            self.val[r], self.col[r] = float(mags[k]), k

    def best(self):
        rows = np.flatnonzero(self.val >= 0.0)
        if rows.size == 0:
            return None
        k = rows[np.lexsort((rows, self.col[rows], -self.val[rows]))[0]]
        if self.val[k] == 0.0:
            return None
        return int(self.col[k]), int(k), float(self.val[k])

    def after_rotation(self, i: int, j: int) -> None:
        n = self.h.shape[0]
        redo = {i, j}
        for c in (i, j):
            xs = np.arange(c + 1, n)
            xs = xs[(xs != i) & (xs != j)]
            if xs.size == 0:
                continue
            stale = (self.col[xs] == i) | (self.col[xs] == j)
            redo.update(int(x) for x in xs[stale])
            xs = xs[~stale]
            if self.mask is not None:
                xs = xs[self.mask[xs] != self.mask[c]]
            new = np.abs(self.h[xs, c])
            better = (new > self.val[xs]) | ((new == self.val[xs]) & (c < self.col[xs]))
            upd = xs[better]
            self.val[upd] = new[better]
            self.col[upd] = c
        for r in sorted(redo):
            self.rescan(r)


def run_incremental(h0: np.ndarray, target=None, *, tol: float, max_iter=None, track_unitary=False):
    """Same contract and bits as run_full_scan, O(N) selection per step."""
    h = np.array(h0, dtype=np.complex128, copy=True)
    n = h.shape[0]
    if max_iter is None:
        max_iter = 20 * n * n
    threshold = tol * max_abs(h)
    rm = _RowMax(h, _mask(n, target))
    u = np.eye(n, dtype=np.complex128) if track_unitary else None
    pivots = []
    while True:
        pick = rm.best()
        if pick is None or pick[2] < threshold:
            converged = True
            break
        if len(pivots) >= max_iter:
            converged = False
            break
        i, j, _ = pick
        c, sh, ph, _ = rotation_scalars(h, i, j)
        s = block_s(sh, ph)
        rotate(h, i, j, c, s)
        if u is not None:
            rotate_unitary(u, i, j, c, s)
        rm.after_rotation(i, j)
        pivots.append((i, j))
    return dict(h=h, applied=len(pivots), converged=converged, pivots=np.asarray(pivots, dtype=np.int64).reshape(-1, 2),
                u=u)


def eliminate_pairs(h0: np.ndarray, pairs, u0=None):
    """eliminate_couplings (npad.py:274-297): scalars from the input, applied
    in list order."""
    h = np.array(h0, dtype=np.complex128, copy=True)
    u = None if u0 is None else np.array(u0, dtype=np.complex128, copy=True)
    scal = [rotation_scalars(h, i, j) for i, j in pairs]
    for (i, j), (c, sh, ph, _) in zip(pairs, scal):
        s = block_s(sh, ph)
        rotate(h, i, j, c, s)
        if u is not None:
            rotate_unitary(u, i, j, c, s)
    return h, u


# ---------------------------------------------------------------------------
# Sparse CSR rotation (npad.py:148-232): the restatement the GPU sparse path
# is checked against (and pinned to the reference by tests/golden/npad_sparse.npz).

def _csr_entry(m, r: int, c: int) -> complex:
    """HermitianOperator.entry on CSR (operators.py:101-102)."""
    lo, hi = m.indptr[r], m.indptr[r + 1]
    cols = m.indices[lo:hi]
    pos = int(np.searchsorted(cols, c))
    if pos < cols.size and cols[pos] == c:
        return complex(m.data[lo + pos])
    return 0j


def sparse_rotation_scalars(m, i: int, j: int):
    """givens_rotation_matrix (npad.py:101-123) on a CSR operator."""
    v = _csr_entry(m, j, i)
    g = abs(v)
    phase = float(np.angle(v))
    delta = (_csr_entry(m, i, i).real - _csr_entry(m, j, j).real) / 2.0
    radius = math.hypot(delta, g)
    sign = 1.0 if delta >= 0.0 else -1.0
    cos_t = abs(delta) / radius
    sin_t = sign * g / radius
    cos_half = math.sqrt((1.0 + cos_t) / 2.0)
    return cos_half, sin_t / (2.0 * cos_half), phase, delta == 0.0


def _row_combination(m, i, j, wi, wj):
    """npad.py:148-159."""
    ci = m.indices[m.indptr[i]:m.indptr[i + 1]]
    vi = m.data[m.indptr[i]:m.indptr[i + 1]]
    cj = m.indices[m.indptr[j]:m.indptr[j + 1]]
    vj = m.data[m.indptr[j]:m.indptr[j + 1]]
    cols = np.concatenate([ci, cj])
    vals = np.concatenate([wi * vi, wj * vj])
    uniq, inv = np.unique(cols, return_inverse=True)
    acc = np.zeros(uniq.size, dtype=np.complex128)
    np.add.at(acc, inv, vals)
    return uniq, acc


def _get_at(cols, vals, k) -> complex:
    pos = np.searchsorted(cols, k)
    if pos < cols.size and cols[pos] == k:
        return complex(vals[pos])
    return 0.0


def _set_at(cols, vals, k, value):
    pos = int(np.searchsorted(cols, k))
    if pos < cols.size and cols[pos] == k:
        vals[pos] = value
        return cols, vals
    return np.insert(cols, pos, k), np.insert(vals, pos, value)


def conjugate_sparse(m, i: int, j: int, cos_half: float, sin_half: float, phase: float, max_abs: float):
    """_conjugate_sparse (npad.py:178-232), statement by statement: the new
    CSR after U H U^dag on rows/columns i < j, fill-in below 1e-15 * max|H|
    dropped (npad.py:33)."""
    import scipy.sparse as sps

    c, s = cos_half, -sin_half * np.exp(1j * phase)  # _block_params (npad.py:126-128)
    ca, va = _row_combination(m, i, j, c, -np.conj(s))
    cb, vb = _row_combination(m, i, j, s, c)
    ai, aj = _get_at(ca, va, i), _get_at(ca, va, j)
    bi, bj = _get_at(cb, vb, i), _get_at(cb, vb, j)
    new_ai = (c * ai - s * aj).real
    new_aj = np.conj(s) * ai + c * aj
    new_bj = (np.conj(s) * bi + c * bj).real
    ca, va = _set_at(ca, va, i, new_ai)
    ca, va = _set_at(ca, va, j, new_aj)
    cb, vb = _set_at(cb, vb, i, np.conj(new_aj))
    cb, vb = _set_at(cb, vb, j, new_bj)
    drop = 1e-15 * max_abs
    keep_a = np.abs(va) > drop
    keep_b = np.abs(vb) > drop
    ca, va = ca[keep_a], va[keep_a]
    cb, vb = cb[keep_b], vb[keep_b]
    data = m.data.copy()
    data[m.indptr[i]:m.indptr[i + 1]] = 0
    data[m.indptr[j]:m.indptr[j + 1]] = 0
    data[np.isin(m.indices, (i, j))] = 0
    base = sps.csr_matrix((data, m.indices.copy(), m.indptr.copy()), shape=m.shape)
    other_a = (ca != i) & (ca != j)
    other_b = (cb != i) & (cb != j)
    rows = np.concatenate([np.full(ca.size, i, dtype=np.int64), np.full(cb.size, j, dtype=np.int64),
                           ca[other_a].astype(np.int64), cb[other_b].astype(np.int64)])
    cols = np.concatenate([ca.astype(np.int64), cb.astype(np.int64), np.full(int(other_a.sum()), i, dtype=np.int64),
                           np.full(int(other_b.sum()), j, dtype=np.int64)])
    vals = np.concatenate([va, vb, np.conj(va[other_a]), np.conj(vb[other_b])])
    delta = sps.csr_matrix((vals, (rows, cols)), shape=m.shape)
    out = base + delta
    out.eliminate_zeros()
    out.sort_indices()
    return out


def eliminate_sparse(m, i: int, j: int):
    """eliminate_coupling (npad.py:262-271) on a CSR operator."""
    max_abs = float(np.max(np.abs(m.data))) if m.nnz else 0.0
    ch, sh, ph, _ = sparse_rotation_scalars(m, i, j)
    return conjugate_sparse(m, i, j, ch, sh, ph, max_abs)
