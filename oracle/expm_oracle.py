"""exp(-iH) restatement (reference expm.py:40-71), numpy."""
from __future__ import annotations

import numpy as np

TAYLOR_ORDER = 18  # expm.py:19
SCALE_TARGET = 0.5  # expm.py:20


def expm_minus_i(h: np.ndarray) -> np.ndarray:
    """_expm_minus_i (expm.py:56-71): scale to max-row-sum <= 0.5, Taylor to
    order 18, square back."""
    a = -1j * np.asarray(h, dtype=np.complex128)
    n = a.shape[0]
    norm = float(np.max(np.abs(a).sum(axis=1))) if n else 0.0
    squarings = 0
    if norm > SCALE_TARGET:
        squarings = int(np.ceil(np.log2(norm / SCALE_TARGET)))
        a = a / (2.0**squarings)
    series = np.eye(n, dtype=np.complex128)
    term = np.eye(n, dtype=np.complex128)
    for k in range(1, TAYLOR_ORDER + 1):
        term = term @ a / k
        series = series + term
    for _ in range(squarings):
        series = series @ series
    return series


def unitarity_defect(u: np.ndarray) -> float:
    """expm.py:35-38."""
    return float(np.linalg.norm(u @ u.conj().T - np.eye(u.shape[0])))


def is_valid_propagator(u: np.ndarray) -> bool:
    """UnitaryPropagator.validate (expm.py:40-47) as a predicate."""
    if unitarity_defect(u) > 1e-10 * u.shape[0]:
        return False
    return abs(abs(np.linalg.det(u)) - 1.0) <= 1e-8
