"""Generate tests/golden/*.npz by running THE REFERENCE ITSELF.

Run in the build container (the reference does not exist on the GPU box):
    python oracle/gen_golden.py [--ref /root/reference/pkg/src]

The reference package is imported read-only from its source tree; the pivot
sequence is captured by wrapping effham.npad.eliminate_coupling in this
harness (npad_run resolves the name at call time, npad.py:354).  Inputs come
from the product's host-side builders (plain numpy), so tests can rebuild
them bit-identically.  Outputs are small (a few MB total).
"""
from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"


def _import_reference(path: str):
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    sys.path.insert(0, path)
    import effham  # noqa: F401

    return sys.modules["effham"]


def _logged_run(effham, op, target=None, **kw):
    log = []
    orig = effham.npad.eliminate_coupling

    def wrapped(state, i, j):
        log.append((i, j))
        return orig(state, i, j)

    effham.npad.eliminate_coupling = wrapped
    try:
        st = effham.npad.npad_run(op, target, **kw)
    finally:
        effham.npad.eliminate_coupling = orig
    return st, np.asarray(log, dtype=np.int64).reshape(-1, 2)


def random_hermitian(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return (a + a.conj().T) / 2.0


def sparse_cases(eff) -> None:
    """10. Sparse CSR rotations (npad.py:148-232): the bench_givens ladder
    (experiments.py:420-453), a sparse npad_run chain (pivot log + every
    intermediate operator is replayable), and a fill-in drop case."""
    import scipy.sparse as sps

    out = {}
    # (a) ladder a^dag a + (a + a^dag), N = 1000, the smallest coupling (0, 1)
    lad = eff.ladder_test_hamiltonian(1000)
    r = eff.eliminate_coupling(eff.NPADState.from_operator(lad), 0, 1).current.data
    out.update(lad_indptr=lad.data.indptr, lad_indices=lad.data.indices, lad_data=lad.data.data,
               lad_out_indptr=r.indptr, lad_out_indices=r.indices, lad_out_data=r.data)
    # (b) random sparse Hermitian (bitwise), greedy npad_run for 40 rotations
    rng = np.random.default_rng(5)
    n = 200
    a = sps.random(n, n, density=0.03, random_state=rng, dtype=np.complex128, data_rvs=lambda k: rng.standard_normal(k)
                   + 1j * rng.standard_normal(k), format="csr")
    h = sps.triu(a + a.conj().T, k=1)
    h = (h + h.conj().T + sps.diags(np.linspace(0.0, 5.0, n))).tocsr().astype(np.complex128)
    h.sum_duplicates()
    h.sort_indices()
    op = eff.HermitianOperator(h)
    st, piv = _logged_run(eff, op, tol=1e-12, max_iter=40)
    fin = st.current.data
    out.update(rnd_indptr=h.indptr, rnd_indices=h.indices, rnd_data=h.data, rnd_pivots=piv,
               rnd_out_indptr=fin.indptr, rnd_out_indices=fin.indices, rnd_out_data=fin.data)
    # (c) exact cancellation: rows (p, q) of level 2 aligned with an eigenvector
    # of the (0, 1) block, so one new coupling falls under the drop threshold
    blk = np.array([[1.0, 0.3 - 0.4j], [0.3 + 0.4j, -0.5]])
    w, vecs = np.linalg.eigh(blk)
    pq = 0.7 * vecs[:, 0].conj()
    dense = np.zeros((3, 3), dtype=complex)
    dense[:2, :2] = blk
    dense[2, 2] = 2.0
    dense[0, 2], dense[1, 2] = pq[0], pq[1]
    dense[2, 0], dense[2, 1] = np.conj(pq[0]), np.conj(pq[1])
    hc = sps.csr_matrix(dense)
    rc = eff.eliminate_coupling(eff.NPADState.from_operator(eff.HermitianOperator(hc, validate=False)), 0, 1)
    rc = rc.current.data
    out.update(can_dense=dense, can_out_indptr=rc.indptr, can_out_indices=rc.indices, can_out_data=rc.data)
    np.savez_compressed(GOLD / "npad_sparse.npz", **out)
    print("sparse: ladder nnz", lad.data.nnz, "->", r.nnz, "; random", h.nnz, "->", fin.nnz, "applied", st.applied,
          "; cancel", hc.nnz, "->", rc.nnz)


def experiment_cases(eff) -> None:
    """11. The reference's experiment runners (experiments.py:233-411) on small
    configs: JCH Mott lobes, driven qubit, spin-chain trajectory and error
    sweep.  Wall-time columns are not produced by these modes."""
    import importlib

    ex = importlib.import_module("effham.experiments")
    out = {}
    cases = {
        "jch": (ex.run_jch_mott, ex.JchMottConfig, dict(n_lobes=2, grid_points=7, n_max=5)),
        "qubit": (ex.run_driven_qubit, ex.DrivenQubitConfig,
                  dict(t_final=20.0, samples=4001, m_magnus=20, m_reference=400)),
        "qubit_sin2": (ex.run_driven_qubit, ex.DrivenQubitConfig,
                       dict(envelope="sin2", drive_ratio=0.5, t_final=30.0, samples=6001, m_magnus=30,
                            m_reference=600)),
        "chain_traj": (ex.run_spin_chain, ex.SpinChainConfig,
                       dict(mode="trajectory", length=5, samples=4001, m_magnus=40, rk_steps=100)),
        "chain_sweep": (ex.run_spin_chain, ex.SpinChainConfig,
                        dict(mode="error-sweep", length=4, samples=3201, sweep_m=[5, 10, 20], m_reference=160,
                             sweep_rk=[100, 200], rk_reference=800)),
    }
    for name, (fn, cls, cfgd) in cases.items():
        fields, rows = fn(ex.config_from_dict(cls, cfgd))
        for f in fields:
            vals = [r[f] for r in rows]
            out[f"{name}__{f}"] = np.array(vals)
        out[f"{name}__cfg"] = np.array(repr(cfgd))
        print("experiments:", name, len(rows), "rows")
    np.savez_compressed(GOLD / "experiments.npz", **out)


def large_cases(eff) -> None:
    """12. The reference itself at the BASELINE sizes: config 4 sweep points
    (dim 1024, subspace mode, to convergence) and the first rotations of
    config 3 (dim 4096, full mode).  Stored: pivots, counts, the final
    diagonal and a few final rows (the full matrices are 16 / 256 MiB)."""
    sys.path.insert(0, str(ROOT))
    from paper_2411_09982_b200 import models as M

    out = {}
    pts = M.sweep_points(32, 32)
    tgt = M.sweep_target(256)
    for k, idx in enumerate((0, 31, 1023)):
        wq, al, wr, g = pts[idx]
        h = M.transmon_resonator_hamiltonian(4, 256, omega_q=wq, alpha=al, omega_r=wr, g=g).data
        st, piv = _logged_run(eff, eff.HermitianOperator(h), tgt, tol=1e-12)
        fin = st.current.data
        out[f"sweep{k}_point"] = pts[idx]
        out[f"sweep{k}_pivots"] = piv
        out[f"sweep{k}_applied"] = st.applied
        out[f"sweep{k}_converged"] = st.converged
        out[f"sweep{k}_diag"] = np.real(np.diag(fin)).copy()
        out[f"sweep{k}_rows"] = fin[[0, 4, 256, 700]].copy()
        print("sweep point", idx, st.applied, st.converged, flush=True)
    h = M.transmon_resonator_hamiltonian(4, 1024).data
    st, piv = _logged_run(eff, eff.HermitianOperator(h), tol=1e-12, max_iter=60)
    fin = st.current.data
    out["c3_pivots"] = piv
    out["c3_applied"] = st.applied
    out["c3_diag"] = np.real(np.diag(fin)).copy()
    rows = sorted({int(r) for r in piv.ravel()[:6]} | {0, 4095})
    out["c3_rows_idx"] = np.array(rows)
    out["c3_rows"] = fin[rows].copy()
    print("config 3 first", st.applied, "rotations", flush=True)
    np.savez_compressed(GOLD / "npad_large_ref.npz", **out)

    # config 2 at full size, order 1 (the reference has no second order):
    # every 1000th trajectory row and the last one
    ch, grid = M.driven_transmon(3, intervals=100_000, sub=4)
    rch = eff.ControlledHamiltonian(eff.HermitianOperator(ch.drift.data),
                                    [eff.HermitianOperator(c.data) for c in ch.controls])
    rgrid = eff.ControlGrid(grid.t_start, grid.t_end, grid.signals)
    tr = eff.evolve(rch, rgrid, 100_000, np.array([1, 0, 0], dtype=complex), check=False)
    np.savez_compressed(GOLD / "magnus_config2_order1_ref.npz", rows=tr.amplitudes[::1000].copy(),
                        last=tr.amplitudes[-1].copy(), times=tr.times[::1000].copy())
    print("config 2 order 1 reference trajectory sampled", flush=True)

    # config 5 (12-spin Heisenberg chain, dim 4096): the first 2 of its 4096
    # intervals, order 1 (36.7 s per interval on the reference)
    ch5 = M.heisenberg_chain_hamiltonians(12)
    full = M.synthetic_transfer_pulse(25.0, 4096 * 8 + 1, seed=7)
    sig5 = full.signals[:, : 2 * 8 + 1]
    rch5 = eff.ControlledHamiltonian(eff.HermitianOperator(ch5.drift.data),
                                     [eff.HermitianOperator(c.data) for c in ch5.controls])
    rgrid5 = eff.ControlGrid(0.0, 25.0 * 2 / 4096, sig5)
    psi5 = np.zeros(4096, dtype=complex)
    psi5[0] = 1.0
    tr5 = eff.evolve(rch5, rgrid5, 2, psi5, check=False)
    np.savez_compressed(GOLD / "magnus_config5_first2_ref.npz", traj=tr5.amplitudes, signals=sig5,
                        t_end=25.0 * 2 / 4096)
    print("config 5 first 2 intervals", flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--only", default=None,
                    help="'sparse' / 'experiments' / 'large': regenerate only those vectors")
    args = ap.parse_args()
    eff = _import_reference(args.ref)
    sys.path.insert(0, str(ROOT))
    from paper_2411_09982_b200 import models as M  # host builders only (numpy)

    GOLD.mkdir(parents=True, exist_ok=True)
    if args.only == "sparse":
        sparse_cases(eff)
        return
    if args.only == "experiments":
        experiment_cases(eff)
        return
    if args.only == "large":
        large_cases(eff)
        return

    # 1. NPAD config 1: transmon 3 x resonator 20, full mode, tol 1e-12
    h = M.transmon_resonator_hamiltonian(3, 20).data
    st, piv = _logged_run(eff, eff.HermitianOperator(h), tol=1e-12)
    np.savez_compressed(GOLD / "npad_tr3x20_full.npz", h=h, pivots=piv, final=st.current.data,
                        applied=st.applied, converged=st.converged, tol=1e-12)
    print("tr3x20", st.applied, st.converged)

    # 2. random complex Hermitian, full mode, with unitary tracking
    h = random_hermitian(24, 7)
    st, piv = _logged_run(eff, eff.HermitianOperator(h), tol=1e-12, track_unitary=True)
    np.savez_compressed(GOLD / "npad_rand24_full_u.npz", h=h, pivots=piv, final=st.current.data,
                        applied=st.applied, converged=st.converged, u=st.accumulated_unitary, tol=1e-12)
    print("rand24", st.applied, st.converged)

    # 3. subspace mode on 4 x 30
    h = M.transmon_resonator_hamiltonian(4, 30, omega_q=6.2, g=0.15).data
    tgt = M.sweep_target(30)
    st, piv = _logged_run(eff, eff.HermitianOperator(h), tgt, tol=1e-12)
    np.savez_compressed(GOLD / "npad_tr4x30_sub.npz", h=h, pivots=piv, final=st.current.data, target=np.array(tgt),
                        applied=st.applied, converged=st.converged, tol=1e-12)
    print("tr4x30 sub", st.applied, st.converged)

    # 4. max_iter truncation on 4 x 60 (dim 240)
    h = M.transmon_resonator_hamiltonian(4, 60).data
    st, piv = _logged_run(eff, eff.HermitianOperator(h), tol=1e-12, max_iter=150)
    np.savez_compressed(GOLD / "npad_tr4x60_k150.npz", h=h, pivots=piv, final=st.current.data,
                        applied=st.applied, converged=st.converged, tol=1e-12, max_iter=150)
    print("tr4x60 k150", st.applied, st.converged)

    # 5. eliminate_couplings on the JC site (Mott pairs), dense input
    p = eff.JCSiteParams(omega=1.0, qubit_freq=0.8, g=0.1, mu=0.3, n_max=8)
    hjc = eff.jc_onsite_hamiltonian(p).to_dense()
    pairs = [(2 * m - 1, 2 * m) for m in range(1, 6)]
    st = eff.eliminate_couplings(eff.NPADState.from_operator(eff.HermitianOperator(hjc), track_unitary=True), pairs)
    np.savez_compressed(GOLD / "npad_jc_pairs.npz", h=hjc, pairs=np.array(pairs), final=st.current.data,
                        u=st.accumulated_unitary, applied=st.applied)

    # 6. AC1: 1000 random 2-level rotations (givens scalars)
    rng = np.random.default_rng(11)
    eps = rng.uniform(-2, 2, 1000)
    dl = rng.uniform(-1, 1, 1000)
    dl[:20] = 0.0  # degenerate cases
    g = rng.uniform(1e-3, 1, 1000)
    phi = rng.uniform(-np.pi, np.pi, 1000)
    mats = np.empty((1000, 2, 2), dtype=np.complex128)
    rows = np.empty((1000, 4))
    after = np.empty((1000, 2, 2), dtype=np.complex128)
    for k in range(1000):
        m2 = np.array([[eps[k] + dl[k], g[k] * np.exp(-1j * phi[k])], [g[k] * np.exp(1j * phi[k]), eps[k] - dl[k]]])
        mats[k] = m2
        op = eff.HermitianOperator(m2)
        rot = eff.givens_rotation_matrix(op, 0, 1)
        rows[k] = (rot.cos_half, rot.sin_half, rot.phase, float(rot.degenerate))
        after[k] = eff.unitary_transformation(op, rot).data
    np.savez_compressed(GOLD / "givens_2x2.npz", mats=mats, params=rows, after=after)

    # 7. expm on random Hermitian matrices of several sizes
    hs = {f"h{n}": random_hermitian(n, 100 + n) * s for n, s in [(3, 0.1), (3, 3.0), (8, 0.7), (40, 0.05), (64, 2.0)]}
    us = {k.replace("h", "u"): eff.expm_unitary(v).entries for k, v in hs.items()}
    np.savez_compressed(GOLD / "expm.npz", **hs, **us)

    # 8. Magnus order 1: driven transmon (config-2 family), M = 2000, sub = 4
    ch, grid = M.driven_transmon(3, intervals=2000, sub=4)
    d0 = ch.drift.data
    ctr = np.stack([c.data for c in ch.controls])
    ref_ch = eff.ControlledHamiltonian(eff.HermitianOperator(d0), [eff.HermitianOperator(c) for c in ctr])
    ref_grid = eff.ControlGrid(grid.t_start, grid.t_end, grid.signals)
    psi0 = np.zeros(3, dtype=np.complex128)
    psi0[0] = 1
    iv = eff.magnus_intervals(ref_ch, ref_grid, 2000)
    traj, props = eff.evolve(ref_ch, ref_grid, 2000, psi0, return_propagators=True, check=True)
    np.savez_compressed(GOLD / "magnus_transmon_m2000.npz", drift=d0, controls=ctr, signals=grid.signals,
                        t=np.array([grid.t_start, grid.t_end]), m=2000, psi0=psi0, coeffs=iv.coefficients,
                        hbar_head=np.stack([iv.effective_hams[k].data for k in range(16)]),
                        u_head=np.stack([props[k].entries for k in range(16)]), traj=traj.amplitudes)

    # 9. Magnus order 1 on the reference spin chain (L = 6, M = 20, sub = 8)
    pc = eff.SpinChainParams(length=6, qubit_freq=1.0, j_nn=0.25, g_nnn=0.05)
    ch6 = eff.spin_chain_hamiltonians(pc)
    grid6 = eff.synthetic_transfer_pulse(25.0, 20 * 8 + 1, seed=3)
    psi6 = np.zeros(64, dtype=np.complex128)
    psi6[0] = 1
    traj6 = eff.evolve(ch6, grid6, 20, psi6, check=True)
    np.savez_compressed(GOLD / "magnus_spin6_m20.npz", drift=ch6.drift.to_dense(),
                        controls=np.stack([c.to_dense() for c in ch6.controls]), signals=grid6.signals,
                        t=np.array([grid6.t_start, grid6.t_end]), m=20, psi0=psi6, traj=traj6.amplitudes,
                        coeffs=eff.magnus_coefficients(grid6, 20))
    sparse_cases(eff)
    experiment_cases(eff)
    print("wrote", sorted(p.name for p in GOLD.glob("*.npz")))


if __name__ == "__main__":
    main()
