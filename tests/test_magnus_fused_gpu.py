"""Single-pass fused Magnus kernel (N <= 4) and the host-buffer pipeline
(qch_magnus_evolve_host_c128) vs the oracle, at BASELINE config-2 size and at
tile / chunk boundaries.  Bar: 1e-10 relative Frobenius (north star)."""
import numpy as np
import pytest

from conftest import rel_fro
from oracle import magnus_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


def _oracle(ch, grid, m, psi0, order):
    d0 = ch.drift.data
    ctr = np.stack([c.data for c in ch.controls]) if ch.controls else np.zeros((0,) + d0.shape, complex)
    return magnus_oracle.evolve(d0, ctr, grid.signals, grid.t_start, grid.t_end, m, psi0, order=order)


def test_config2_full_size_vs_oracle(E):
    # BASELINE config 2: driven 3-level transmon, 1e5 intervals, order 2
    m = 100_000
    ch, grid = E.driven_transmon(3, intervals=m, sub=4)
    psi0 = np.array([1, 0, 0], dtype=complex)
    got = E.evolve(ch, grid, m, psi0, order=2, check=True)
    ref = _oracle(ch, grid, m, psi0, 2)
    assert got.amplitudes.shape == (m + 1, 3)
    assert rel_fro(got.amplitudes, ref) <= 1e-10
    np.testing.assert_array_equal(got.times, np.linspace(grid.t_start, grid.t_end, m + 1))
    # size-independent property: every state normalised
    assert np.abs(np.linalg.norm(got.amplitudes, axis=1) - 1).max() < 1e-12


@pytest.mark.parametrize("m", [1, 2, 63, 64, 65, 129, 3 * 16384 + 17])
@pytest.mark.parametrize("order", [1, 2])
def test_host_and_device_paths_vs_oracle(E, m, order):
    ch, grid = E.driven_transmon(3, intervals=m, sub=4, t_final=100.0 * m / 100_000 + 1.0)
    psi0 = np.array([0.6, 0.8j, 0], dtype=complex)
    ref = _oracle(ch, grid, m, psi0, order)
    host = E.evolve(ch, grid, m, psi0, order=order)
    assert rel_fro(host.amplitudes, ref) <= 1e-10
    import torch

    dev = E.magnus.evolve_device(ch, grid, m, torch.tensor(psi0, device="cuda"), order=order)
    assert rel_fro(dev.cpu().numpy(), ref) <= 1e-10


def test_many_chunks_and_pageable_signals(E):
    m = 8 * 16384 + 5  # 8 pipeline chunks, ragged last tile
    ch, grid = E.driven_transmon(3, intervals=m, sub=4)
    sig = np.array(grid.signals, order="C")  # plain pageable numpy
    grid2 = E.ControlGrid(grid.t_start, grid.t_end, sig)
    psi0 = np.array([1, 0, 0], dtype=complex)
    got = E.evolve(ch, grid2, m, psi0, order=2)
    ref = _oracle(ch, grid2, m, psi0, 2)
    assert rel_fro(got.amplitudes, ref) <= 1e-10


@pytest.mark.parametrize("n", [1, 2, 4])
def test_other_small_dims(E, n):
    rng = np.random.default_rng(n)

    def herm(scale):
        a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        return (a + a.conj().T) * scale

    ch = E.ControlledHamiltonian(E.HermitianOperator(herm(0.5)), [E.HermitianOperator(herm(0.3)) for _ in range(3)])
    m, sub = 2000, 3
    sig = rng.standard_normal((3, m * sub + 1))
    grid = E.ControlGrid(0.0, 40.0, sig)
    psi0 = np.zeros(n, complex)
    psi0[0] = 1
    for order in (1, 2):
        got = E.evolve(ch, grid, m, psi0, order=order)
        assert rel_fro(got.amplitudes, _oracle(ch, grid, m, psi0, order)) <= 1e-10


def test_no_controls_constant_hamiltonian(E):
    h = np.diag([0.0, 1.0, 2.5]).astype(complex)
    ch = E.ControlledHamiltonian(E.HermitianOperator(h), [])
    grid = E.ControlGrid(0.0, 3.0, samples=301)
    psi0 = np.ones(3, complex) / np.sqrt(3)
    got = E.evolve(ch, grid, 100, psi0, order=2)
    t = np.linspace(0, 3, 101)
    exact = np.exp(-1j * np.outer(t, np.diag(h).real)) * psi0
    assert rel_fro(got.amplitudes, exact) <= 1e-12


def test_return_propagators_matches_oracle(E):
    m = 300
    ch, grid = E.driven_transmon(3, intervals=m, sub=4, t_final=7.0)
    psi0 = np.array([1, 0, 0], dtype=complex)
    traj, props = E.evolve(ch, grid, m, psi0, order=2, return_propagators=True)
    hb = magnus_oracle.effective_hamiltonians(ch.drift.data, np.stack([c.data for c in ch.controls]), grid.signals,
                                              grid.t_start, grid.t_end, m, order=2)
    from oracle import expm_oracle

    want = np.stack([expm_oracle.expm_minus_i(h) for h in hb])
    assert rel_fro(np.stack([p.entries for p in props]), want) <= 1e-12
    assert rel_fro(traj.amplitudes, _oracle(ch, grid, m, psi0, 2)) <= 1e-10


def test_errors_through_host_path(E):
    ch, grid = E.driven_transmon(3, intervals=100, sub=4, t_final=10.0)
    psi0 = np.array([1, 0, 0], dtype=complex)
    # non-Hermitian drift -> non-unitary propagators
    bad = ch.drift.data.copy()
    bad[1, 1] += 0.5j
    chb = E.ControlledHamiltonian(E.HermitianOperator(bad, validate=False), ch.controls)
    with pytest.raises(E.NonFinite):
        E.evolve(chb, grid, 100, psi0, check=True)
    with pytest.raises(E.NormDrift):
        E.evolve(chb, grid, 100, psi0, check=False)
    with pytest.raises(E.GridMismatch):
        E.evolve(ch, grid, 7, psi0)
    nan = ch.drift.data.copy()
    nan[0, 0] = np.nan
    with pytest.raises(E.NonFinite):
        E.evolve(E.ControlledHamiltonian(E.HermitianOperator(nan, validate=False), ch.controls), grid, 100, psi0)


def test_evolve_plan_replay(E):
    m = 4096
    ch, grid = E.driven_transmon(3, intervals=m, sub=4, t_final=20.0)
    psi0 = np.array([1, 0, 0], dtype=complex)
    plan = E.EvolvePlan(ch, grid, m, psi0, order=2, check=True)
    for _ in range(3):
        out = plan.run()
    plan.check()
    ref = _oracle(ch, grid, m, psi0, 2)
    assert rel_fro(out.cpu().numpy(), ref) <= 1e-10
    # new signals in place, replay again
    sig2 = grid.signals * 0.5
    plan.set_signals(sig2)
    out2 = plan.run().cpu().numpy()
    ref2 = _oracle(ch, E.ControlGrid(grid.t_start, grid.t_end, sig2), m, psi0, 2)
    assert rel_fro(out2, ref2) <= 1e-10


@pytest.mark.parametrize("mode", ["map", "copy", "stream"])
def test_host_call_signal_modes(E, mode, monkeypatch):
    # page-locked signals: zero-copy (default), copy-engine H2D, or chunked
    # copy-engine stream polled by the running kernel — same results
    import torch

    m = 20_000
    ch, grid = E.driven_transmon(3, intervals=m, sub=4, t_final=20.0)
    pinned = torch.empty(grid.signals.shape, dtype=torch.float64).pin_memory()
    pinned.numpy()[:] = grid.signals
    g2 = E.ControlGrid(grid.t_start, grid.t_end, pinned.numpy())
    psi0 = np.array([1, 0, 0], dtype=complex)
    monkeypatch.setenv("QCH_SIG_MODE", mode)
    got = E.evolve(ch, g2, m, psi0, order=2)
    assert rel_fro(got.amplitudes, _oracle(ch, grid, m, psi0, 2)) <= 1e-10


def test_evolve_plan_flags_every_replay(E):
    # the plan's self-cleaning workspace: status words are recomputed on every
    # replay (the kernel's last block resets them), a bad plan keeps raising
    m = 2048
    ch, grid = E.driven_transmon(3, intervals=m, sub=4, t_final=10.0)
    bad = ch.drift.data.copy()
    bad[1, 1] += 0.5j
    chb = E.ControlledHamiltonian(E.HermitianOperator(bad, validate=False), ch.controls)
    psi0 = np.array([1, 0, 0], dtype=complex)
    plan = E.EvolvePlan(chb, grid, m, psi0, order=2, check=False)
    for _ in range(3):
        plan.run()
        with pytest.raises(E.NormDrift):
            plan.check()
    good = E.EvolvePlan(ch, grid, m, psi0, order=2, check=True)
    for _ in range(3):
        good.run()
        good.check()


def test_evolve_plan_many_waves(E):
    # more tiles than resident blocks: groups of tiles, look-back over groups,
    # workspace reused across replays
    import torch

    m = 1_000_000
    ch, grid = E.driven_transmon(3, intervals=m, sub=4, t_final=500.0)
    psi0 = np.array([1, 0, 0], dtype=complex)
    plan = E.EvolvePlan(ch, grid, m, psi0, order=2, check=True)
    outs = []
    for _ in range(3):
        outs.append(plan.run().clone())
    plan.check()
    from paper_2411_09982_b200 import magnus as mg

    want = mg.evolve_device(ch, grid, m, torch.tensor(psi0, device="cuda"), check=True, order=2)
    for o in outs:
        assert rel_fro(o.cpu().numpy(), want.cpu().numpy()) <= 1e-12
    sub = 20_000
    ref = _oracle(ch, E.ControlGrid(grid.t_start, grid.t_start + (grid.t_end - grid.t_start) * sub / m,
                                    grid.signals[:, : sub * 4 + 1]), sub, psi0, 2)
    assert rel_fro(outs[-1][: sub + 1].cpu().numpy(), ref) <= 1e-10


def test_host_call_workspace_relayout(E):
    # the host call's cached workspace is re-initialised when (N, M) change
    psi0 = np.array([1, 0, 0], dtype=complex)
    for m in (1000, 3000, 1000, 257, 3000):
        ch, grid = E.driven_transmon(3, intervals=m, sub=4, t_final=10.0)
        got = E.evolve(ch, grid, m, psi0, order=2)
        assert rel_fro(got.amplitudes, _oracle(ch, grid, m, psi0, 2)) <= 1e-10
    ch2, grid2 = E.driven_transmon(2, intervals=500, sub=4, t_final=10.0)
    got = E.evolve(ch2, grid2, 500, np.array([1, 0], dtype=complex), order=1)
    assert rel_fro(got.amplitudes, _oracle(ch2, grid2, 500, np.array([1, 0], dtype=complex), 1)) <= 1e-10


@pytest.mark.parametrize("t0,t1,m", [(0.0, 100.0, 100_000), (-3.7, 12.9, 777), (1e-3, 1e-3 + 1e-9, 1000),
                                     (0.1, 0.7, 3)])
def test_host_call_times_are_linspace(E, t0, t1, m):
    # times come from the C-ABI call (filled on the host during the kernel),
    # bit for bit np.linspace (magnus.py:263)
    ch, grid = E.driven_transmon(3, intervals=m, sub=4, t_final=10.0)
    g2 = E.ControlGrid(t0, t1, grid.signals)
    out = E.evolve(ch, g2, m, np.array([1, 0, 0], dtype=complex), order=1, check=False)
    np.testing.assert_array_equal(out.times, np.linspace(t0, t1, m + 1))


@pytest.mark.parametrize("sub,k", [(1, 2), (2, 1), (4, 1), (8, 2), (16, 2), (5, 3)])
def test_samples_per_interval_and_controls(E, sub, k):
    # the fused kernel's window staging (sub*256+1 samples per control up to
    # 24 KB), the fixed-SUB register path (sub = 4) and the unstaged global
    # path (large windows), for 1-3 controls, orders 1 and 2, host and plan
    rng = np.random.default_rng(100 * sub + k)

    def herm(scale):
        a = rng.standard_normal((3, 3)) + 1j * rng.standard_normal((3, 3))
        return (a + a.conj().T) * scale

    ch = E.ControlledHamiltonian(E.HermitianOperator(herm(0.5)), [E.HermitianOperator(herm(0.2)) for _ in range(k)])
    m = 3001
    grid = E.ControlGrid(0.0, 30.0, np.sin(np.outer(np.arange(1, k + 1), np.linspace(0, 9, m * sub + 1))))
    psi0 = np.array([0.6, 0.8j, 0.0])
    for order in (1, 2):
        ref = _oracle(ch, grid, m, psi0, order)
        got = E.evolve(ch, grid, m, psi0, order=order)
        assert rel_fro(got.amplitudes, ref) <= 1e-10, (sub, k, order)
        plan = E.EvolvePlan(ch, grid, m, psi0, order=order, check=True)
        plan.run()
        plan.check()
        assert rel_fro(plan.run().cpu().numpy(), ref) <= 1e-10, (sub, k, order, "plan")


@pytest.mark.parametrize("m", [1, 2, 255, 256, 257, 8191, 8193])
def test_interval_counts_around_tiles(E, m):
    # partial tiles, single-tile groups, exactly one tile, one group boundary
    ch, grid = E.driven_transmon(3, intervals=m, sub=4, t_final=0.05 * m)
    psi0 = np.array([1, 0, 0], dtype=complex)
    ref = _oracle(ch, grid, m, psi0, 2)
    assert rel_fro(E.evolve(ch, grid, m, psi0, order=2).amplitudes, ref) <= 1e-10
    plan = E.EvolvePlan(ch, grid, m, psi0, order=2, check=True)
    for _ in range(2):
        out = plan.run()
    plan.check()
    assert rel_fro(out.cpu().numpy(), ref) <= 1e-10


def test_config2_full_size_order1_vs_reference_itself(E):
    # BASELINE config 2 workload at order 1 against the reference's own evolve
    # (tests/golden/magnus_config2_order1_ref.npz: every 1000th row)
    from pathlib import Path

    g = np.load(Path(__file__).parent / "golden" / "magnus_config2_order1_ref.npz")
    m = 100_000
    ch, grid = E.driven_transmon(3, intervals=m, sub=4)
    got = E.evolve(ch, grid, m, np.array([1, 0, 0], dtype=complex), order=1, check=False)
    assert rel_fro(got.amplitudes[::1000], g["rows"]) <= 1e-10
    assert rel_fro(got.amplitudes[-1], g["last"]) <= 1e-10
    np.testing.assert_array_equal(got.times[::1000], g["times"])
