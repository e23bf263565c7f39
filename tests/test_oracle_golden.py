"""The CPU oracle (oracle/) against golden vectors produced by the reference
itself (oracle/gen_golden.py).  Bit-exact: same numpy operations, same host."""
import numpy as np
import pytest

from pathlib import Path

from oracle import expm_oracle, magnus_oracle, npad_oracle

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("runner", [npad_oracle.run_full_scan, npad_oracle.run_incremental])
@pytest.mark.parametrize("case", ["npad_tr3x20_full", "npad_rand24_full_u", "npad_tr4x30_sub", "npad_tr4x60_k150"])
def test_npad_oracle_bit_exact(golden, runner, case):
    g = golden(case)
    target = g["target"].tolist() if "target" in g else None
    max_iter = int(g["max_iter"]) if "max_iter" in g else None
    out = runner(g["h"], target, tol=float(g["tol"]), max_iter=max_iter, track_unitary="u" in g)
    assert out["applied"] == int(g["applied"])
    assert out["converged"] == bool(g["converged"])
    np.testing.assert_array_equal(out["pivots"], g["pivots"])
    np.testing.assert_array_equal(out["h"], g["final"])
    if "u" in g:
        np.testing.assert_array_equal(out["u"], g["u"])


def test_eliminate_pairs_oracle(golden):
    g = golden("npad_jc_pairs")
    h, u = npad_oracle.eliminate_pairs(g["h"], [tuple(p) for p in g["pairs"]], np.eye(g["h"].shape[0]))
    np.testing.assert_array_equal(h, g["final"])
    np.testing.assert_array_equal(u, g["u"])


def test_givens_oracle(golden):
    g = golden("givens_2x2")
    for k in range(0, 1000, 7):
        c, sh, ph, deg = npad_oracle.rotation_scalars(g["mats"][k], 0, 1)
        assert (c, sh, ph, float(deg)) == tuple(g["params"][k])
        h = g["mats"][k].copy()
        npad_oracle.rotate(h, 0, 1, c, npad_oracle.block_s(sh, ph))
        np.testing.assert_array_equal(h, g["after"][k])


def test_expm_oracle(golden):
    g = golden("expm")
    for key in [k for k in g if k.startswith("h")]:
        np.testing.assert_array_equal(expm_oracle.expm_minus_i(g[key]), g["u" + key[1:]])


@pytest.mark.parametrize("case", ["magnus_transmon_m2000", "magnus_spin6_m20"])
def test_magnus_oracle(golden, case):
    g = golden(case)
    t0, t1 = g["t"]
    m = int(g["m"])
    c = magnus_oracle.first_order_coefficients(g["signals"], t0, t1, m)
    np.testing.assert_array_equal(c, g["coeffs"])
    traj = magnus_oracle.evolve(g["drift"], g["controls"], g["signals"], t0, t1, m, g["psi0"])
    np.testing.assert_array_equal(traj, g["traj"])
    if "hbar_head" in g:
        hb = magnus_oracle.effective_hamiltonians(g["drift"], g["controls"], g["signals"], t0, t1, m)
        np.testing.assert_array_equal(hb[:16], g["hbar_head"])


def test_sparse_rotation_oracle_bit_exact(golden):
    """The CSR rotation restatement (npad_oracle.conjugate_sparse) against the
    reference's own _conjugate_sparse (npad.py:148-232): same structure, same
    bits."""
    import scipy.sparse as sps

    g = golden("npad_sparse")

    def csr(p, n):
        return sps.csr_matrix((g[p + "_data"], g[p + "_indices"], g[p + "_indptr"]), shape=(n, n))

    def same(a, b):
        np.testing.assert_array_equal(a.indptr, b.indptr)
        np.testing.assert_array_equal(a.indices, b.indices)
        np.testing.assert_array_equal(a.data, b.data)

    n_lad = g["lad_indptr"].size - 1
    same(npad_oracle.eliminate_sparse(csr("lad", n_lad), 0, 1), csr("lad_out", n_lad))
    n = g["rnd_indptr"].size - 1
    m = csr("rnd", n)
    for i, j in g["rnd_pivots"]:
        m = npad_oracle.eliminate_sparse(m, int(i), int(j))
    same(m, csr("rnd_out", n))
    out = npad_oracle.eliminate_sparse(sps.csr_matrix(g["can_dense"]), 0, 1)
    same(out, csr("can_out", 3))


def test_npad_oracle_at_baseline_sizes(golden):
    # the oracle against the reference itself at config-4 / config-3 sizes
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2411_09982_b200 import models as M

    g = golden("npad_large_ref")
    tgt = M.sweep_target(256)
    k = 0  # the 148-rotation point (the others: tests/test_npad_large_ref_gpu.py)
    wq, al, wr, gg = g[f"sweep{k}_point"]
    h = M.transmon_resonator_hamiltonian(4, 256, omega_q=wq, alpha=al, omega_r=wr, g=gg).data
    ref = npad_oracle.run_incremental(h, tgt, tol=1e-12)
    np.testing.assert_array_equal(ref["pivots"], g[f"sweep{k}_pivots"])
    np.testing.assert_array_equal(np.real(np.diag(ref["h"])), g[f"sweep{k}_diag"])
    h = M.transmon_resonator_hamiltonian(4, 1024).data
    ref = npad_oracle.run_incremental(h, tol=1e-12, max_iter=int(g["c3_applied"]))
    np.testing.assert_array_equal(ref["pivots"], g["c3_pivots"])
    np.testing.assert_array_equal(ref["h"][g["c3_rows_idx"]], g["c3_rows"])


def test_long_config3_golden_starts_with_reference_picks():
    # the oracle-made full-length config-3 golden agrees with the reference's
    # own first 60 picks (the part the reference can produce here)
    g = np.load(GOLD / "npad_large_ref.npz")
    L = np.load(GOLD / "npad_config3_full_oracle.npz")
    np.testing.assert_array_equal(L["pivots"][: len(g["c3_pivots"])].astype(np.int64), g["c3_pivots"])
    assert int(L["applied"]) == 292068 and bool(L["converged"])
