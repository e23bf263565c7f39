"""Magnus restatement (reference magnus.py:151-273) plus the second-order
term the reference lacks (parity UNPINNED by
the reference — checked against nested quadrature instead).

Inputs are plain arrays: drift (N,N), controls (K,N,N), signals (K,S),
t_start, t_end.
"""
from __future__ import annotations

import numpy as np

from .expm_oracle import expm_minus_i

NORM_DRIFT_TOL = 1e-6  # magnus.py:28


def first_order_coefficients(signals: np.ndarray, t_start: float, t_end: float, m: int) -> np.ndarray:
    """magnus_coefficients (magnus.py:151-169): (M, K) composite trapezoid."""
    k, samples = signals.shape
    steps = samples - 1
    sub = steps // m
    dt = (t_end - t_start) / steps
    lo = signals[:, :-1].reshape(k, m, sub)
    hi = signals[:, 1:].reshape(k, m, sub)
    return np.ascontiguousarray(((dt / 2.0) * (lo + hi).sum(axis=2)).T)


def second_order_coefficients(signals: np.ndarray, t_start: float, t_end: float, m: int) -> np.ndarray:
    """(M, K + K(K-1)/2): [alpha_k ..., beta_kl (k<l) ...] with, per interval
    and panel a (h = grid spacing, tau = (h/2)(u_a + u_{a+1}), S(a) the
    running sum of tau before panel a):
      alpha_k  = sum_a [h S_k(a) - a h tau_ak] - (h^2/6) sum_a (u_k,a+1 - u_k,a)
      beta_kl  = sum_a [tau_ak S_l(a) - tau_al S_k(a)]
                 - (h^2/6) sum_a (u_k,a u_l,a+1 - u_l,a u_k,a+1)
    so that X_n = sum_k alpha_k [H0,H_k] + sum_{k<l} beta_kl [H_k,H_l] equals
    the exact double integral of [H(t1), H(t2)] over t2 < t1 in the interval
    for controls linear between samples.  Evaluation order matches
    magnus.cu:interval_coeffs."""
    k, samples = signals.shape
    steps = samples - 1
    sub = steps // m
    h = (t_end - t_start) / steps
    h2 = h / 2.0
    hh6 = (h * h) / 6.0
    ncomm = k + k * (k - 1) // 2
    out = np.zeros((m, ncomm))
    for n in range(m):
        win = signals[:, n * sub:(n + 1) * sub + 1]
        for a in range(k):
            run = acc = lin = 0.0
            for q in range(sub):
                tau = h2 * (win[a, q] + win[a, q + 1])
                acc = acc + (h * run - (float(q) * h) * tau)
                lin = lin + (win[a, q + 1] - win[a, q])
                run = run + tau
            out[n, a] = acc - hh6 * lin
        col = k
        for a in range(k):
            for b in range(a + 1, k):
                sa = sb = acc = cr = 0.0
                for q in range(sub):
                    ta = h2 * (win[a, q] + win[a, q + 1])
                    tb = h2 * (win[b, q] + win[b, q + 1])
                    acc = acc + (ta * sb - tb * sa)
                    cr = cr + (win[a, q] * win[b, q + 1] - win[b, q] * win[a, q + 1])
                    sa = sa + ta
                    sb = sb + tb
                out[n, col] = acc - hh6 * cr
                col += 1
    return out


def commutators(drift: np.ndarray, controls: np.ndarray) -> list[np.ndarray]:
    """[H0,H_k] for each k, then [H_k,H_l] for k < l."""
    ops = []
    k = controls.shape[0]
    for a in range(k):
        ops.append(drift @ controls[a] - controls[a] @ drift)
    for a in range(k):
        for b in range(a + 1, k):
            ops.append(controls[a] @ controls[b] - controls[b] @ controls[a])
    return ops


def effective_hamiltonians(drift, controls, signals, t_start, t_end, m, order=1) -> np.ndarray:
    """assemble_effective_hams (magnus.py:172-190; first order) plus
    (-i/2) X_n for order 2.  Returns (M, N, N)."""
    dt_int = (t_end - t_start) / m
    c1 = first_order_coefficients(signals, t_start, t_end, m) if signals.shape[0] else np.zeros((m, 0))
    out = np.empty((m,) + drift.shape, dtype=np.complex128)
    if order >= 2 and signals.shape[0]:
        c2 = second_order_coefficients(signals, t_start, t_end, m)
        comm = commutators(drift, controls)
    for n in range(m):
        hb = dt_int * drift
        for w, ctrl in zip(c1[n], controls):
            hb = hb + w * ctrl
        if order >= 2 and signals.shape[0]:
            x = np.zeros_like(hb)
            for w, cm in zip(c2[n], comm):
                x = x + w * cm
            hb = hb + (-0.5j) * x
        out[n] = hb
    return out


def evolve(drift, controls, signals, t_start, t_end, m, psi0, order=1, return_propagators=False):
    """evolve dense path (magnus.py:214-267): (M+1, N) trajectory; raises
    RuntimeError('NormDrift n') like _check_norm (magnus.py:270-273)."""
    hams = effective_hamiltonians(drift, controls, signals, t_start, t_end, m, order)
    psi = np.array(psi0, dtype=np.complex128).ravel()
    traj = np.empty((m + 1, psi.size), dtype=np.complex128)
    traj[0] = psi
    props = []
    for n in range(m):
        u = expm_minus_i(hams[n])
        psi = u @ psi
        if abs(float(np.linalg.norm(psi)) - 1.0) > NORM_DRIFT_TOL:
            raise RuntimeError(f"NormDrift {n}")
        traj[n + 1] = psi
        if return_propagators:
            props.append(u)
    if return_propagators:
        return traj, np.asarray(props)
    return traj
