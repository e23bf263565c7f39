"""Long golden vectors from the ORACLE (test infrastructure, build container).

These cases are too long for the reference itself (config 3 to convergence
is ~2 days of effham.npad_run; config 5 order 2 has no reference at all), so
they come from the oracle restatements, which tests/test_oracle_golden.py
pins bit-for-bit to the reference on every case the reference can finish
(incl. the first 60 rotations of this very operator and three config-4
points to convergence).

    python oracle/gen_golden_long.py [--only c3|c5]

c3: npad_oracle.run_incremental on config 3 (transmon 4 x resonator 1024,
    dim 4096, full diagonal, tol 1e-12) to convergence: 292,068 rotations
    (~5 min).  Stored: the whole pivot log as uint16 pairs, applied,
    converged, the final diagonal and a few final rows.
c5: magnus_oracle.evolve ORDER 2 on config 5 (12-spin Heisenberg chain, dim
    4096, synthetic_transfer_pulse(25, 4096*8+1, seed=7)), the first 3 of its
    4096 intervals (reference expm: 18-term Taylor, expm.py:56-71).
c5mid: the same at intervals 2048-2049 (mid-pulse) from a random state.
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def config3_full() -> None:
    from oracle import npad_oracle
    from paper_2411_09982_b200 import models as M  # host numpy builders

    h = M.transmon_resonator_hamiltonian(4, 1024).data
    t0 = time.perf_counter()
    ref = npad_oracle.run_incremental(h, tol=1e-12)
    dt = time.perf_counter() - t0
    piv = ref["pivots"]
    fin = ref["h"]
    rows = sorted({int(r) for r in piv[-3:].ravel()} | {0, 1, 1023, 2048, 4095})
    np.savez_compressed(GOLD / "npad_config3_full_oracle.npz", pivots=piv.astype(np.uint16),
                        applied=ref["applied"], converged=ref["converged"], diag=np.real(np.diag(fin)).copy(),
                        rows_idx=np.array(rows), rows=fin[rows].copy(), seconds=dt)
    print(f"config 3: {ref['applied']} rotations, converged={ref['converged']}, {dt:.0f} s", flush=True)


def config5_order2(n_int: int = 3) -> None:
    from oracle import magnus_oracle
    from paper_2411_09982_b200 import models as M

    ch = M.heisenberg_chain_hamiltonians(12)
    full = M.synthetic_transfer_pulse(25.0, 4096 * 8 + 1, seed=7)
    sig = full.signals[:, : n_int * 8 + 1]
    d0 = ch.drift.to_dense()
    ctr = np.stack([c.to_dense() for c in ch.controls])
    psi0 = np.zeros(4096, dtype=complex)
    psi0[0] = 1.0
    t0 = time.perf_counter()
    traj = magnus_oracle.evolve(d0, ctr, sig, 0.0, 25.0 * n_int / 4096, n_int, psi0, order=2)
    dt = time.perf_counter() - t0
    np.savez_compressed(GOLD / "magnus_config5_order2_oracle.npz", traj=traj, signals=sig,
                        t_end=25.0 * n_int / 4096, seconds=dt)
    print(f"config 5 order 2: {n_int} intervals, {dt:.0f} s", flush=True)


def config5_mid_order2() -> None:
    """Intervals 2048, 2049 of config 5 (mid-pulse, where the second-order
    term matters), order 2, from a fixed random normalised state."""
    from oracle import magnus_oracle
    from paper_2411_09982_b200 import models as M

    ch = M.heisenberg_chain_hamiltonians(12)
    full = M.synthetic_transfer_pulse(25.0, 4096 * 8 + 1, seed=7)
    a, n_int = 2048, 2
    sig = full.signals[:, a * 8: (a + n_int) * 8 + 1]
    t0, t1 = 25.0 * a / 4096, 25.0 * (a + n_int) / 4096
    d0 = ch.drift.to_dense()
    ctr = np.stack([c.to_dense() for c in ch.controls])
    rng = np.random.default_rng(2048)
    psi0 = rng.standard_normal(4096) + 1j * rng.standard_normal(4096)
    psi0 /= np.linalg.norm(psi0)
    tm = time.perf_counter()
    traj = magnus_oracle.evolve(d0, ctr, sig, t0, t1, n_int, psi0, order=2)
    np.savez_compressed(GOLD / "magnus_config5_mid_order2_oracle.npz", traj=traj, signals=sig, t=np.array([t0, t1]))
    print(f"config 5 mid-pulse order 2: {time.perf_counter() - tm:.0f} s", flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None, choices=["c3", "c5", "c5mid"])
    args = ap.parse_args()
    if args.only in (None, "c5"):
        config5_order2()
    if args.only in (None, "c5mid"):
        config5_mid_order2()
    if args.only in (None, "c3"):
        config3_full()


if __name__ == "__main__":
    main()
