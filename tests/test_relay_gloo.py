"""Multi-process (gloo, CPU) tests of the N > 4 Magnus relay
(sharding.evolve_relay): round-robin chunks, the state relayed rank to rank
with send/recv, the error relay, and the trajectory gather.  The per-rank
compute is the CPU oracle injected in place of the GPU kernels; the
distributed result must equal the single-process oracle evolve."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import expm_oracle, magnus_oracle


class OracleRelayCompute:
    """The oracle restatement per chunk (effective Hamiltonians of the chunk's
    signal window, 18-term Taylor expm, sequential product)."""

    def __init__(self, drift_norm_at=None):
        self.drift_norm_at = drift_norm_at  # (chunk start interval, local index): inject a NormDrift

    def setup(self, ch, order):
        self.d0 = ch.drift.to_dense()
        self.ctr = np.stack([c.to_dense() for c in ch.controls])

    def propagators(self, ch, sig, dt, dt_int, m, order, check):
        steps = sig.shape[1] - 1
        hb = magnus_oracle.effective_hamiltonians(self.d0, self.ctr, sig, 0.0, dt * steps, m, order)
        self.start_marker = sig[0, 0]
        return np.stack([expm_oracle.expm_minus_i(h) for h in hb]), None

    def chain(self, us, m, psi_in):
        v = psi_in.numpy()
        rows = []
        for q in range(m):
            v = us[q] @ v
            rows.append(v)
        rows = torch.from_numpy(np.stack(rows))
        if self.drift_norm_at is not None and self.drift_norm_at[0] == self.start_marker:
            return rows, (9, self.drift_norm_at[1], "injected")
        return rows, None

    def to_tensor(self, psi):
        return torch.from_numpy(np.asarray(psi, dtype=complex).copy())

    def empty(self, n):
        return torch.empty(n, dtype=torch.complex128)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(m):
    from paper_2411_09982_b200 import models

    ch = models.heisenberg_chain_hamiltonians(3)  # N = 8
    grid = models.synthetic_transfer_pulse(2.0, m * 4 + 1, seed=5)
    psi0 = np.zeros(8, dtype=complex)
    psi0[0] = 1.0
    return ch, grid, psi0


def _worker(rank, world, port, m, chunk, inject, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_09982_b200 import sharding
        from paper_2411_09982_b200.errors import NormDrift

        ch, grid, psi0 = _problem(m)
        comp = OracleRelayCompute()
        if inject is not None:
            comp.drift_norm_at = (grid.signals[0, inject[0] * 4], inject[1])
        try:
            res = sharding.evolve_relay(ch, grid, m, psi0, order=2, chunk=chunk, compute=comp)
        except NormDrift as e:
            q.put((rank, "NormDrift", str(e)))
            return
        full = res.gather()
        q.put((rank, [(a, b) for a, b, _ in res.chunks], full.numpy()))
    finally:
        dist.destroy_process_group()


def _run(world, m, chunk, inject=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, chunk, inject, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("world,m,chunk", [(2, 12, 2), (2, 9, 4), (3, 10, 1), (3, 7, 3)])
def test_relay_gloo_matches_single_process(world, m, chunk):
    got = _run(world, m, chunk)
    ch, grid, psi0 = _problem(m)
    ref = magnus_oracle.evolve(ch.drift.to_dense(), np.stack([c.to_dense() for c in ch.controls]), grid.signals,
                               grid.t_start, grid.t_end, m, psi0, order=2)
    n_chunks = -(-m // chunk)
    for rank, spans, full in got:
        # round-robin ownership
        assert spans == [(k * chunk, min(m, (k + 1) * chunk)) for k in range(rank, n_chunks, world)]
        np.testing.assert_allclose(full, ref, rtol=0, atol=1e-12)


def test_relay_gloo_error_reaches_every_rank():
    # a NormDrift injected in chunk 2 (intervals 4, 5; rank 0 of 2) at local
    # index 1 -> every rank raises NormDrift for interval 5
    got = _run(2, 12, 2, inject=(4, 1))
    assert [g[1] for g in got] == ["NormDrift", "NormDrift"]
    assert all("interval 5" in g[2] for g in got)


def test_relay_chunk_sizing():
    from paper_2411_09982_b200.sharding import relay_chunk

    assert relay_chunk(4096, 4096, 8) == 16          # 16 x 256 MiB = 4 GiB of propagators
    assert relay_chunk(4096, 4096, 1) == 16
    assert relay_chunk(64, 10, 4) == 3               # at least one chunk per rank
    assert relay_chunk(8, 1, 1) == 1


# -- NPAD sweep sharding (config 4 host logic) ---------------------------------------

class OracleSweepCompute:
    def run(self, points, n_q, n_r, target, tol, max_iter):
        from oracle import npad_oracle
        from paper_2411_09982_b200 import models

        ap, cv, dg = [], [], []
        for wq, al, wr, g in points:
            h = models.transmon_resonator_hamiltonian(n_q, n_r, omega_q=wq, alpha=al, omega_r=wr, g=g).data
            r = npad_oracle.run_incremental(h, target, tol=tol, max_iter=max_iter)
            ap.append(r["applied"])
            cv.append(r["converged"])
            dg.append(np.real(np.diag(r["h"])))
        return (torch.tensor(ap, dtype=torch.int64), torch.tensor(cv, dtype=torch.int32),
                torch.from_numpy(np.stack(dg)), None)


def _sweep_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_09982_b200 import models, sharding

        pts = models.sweep_points(3, 3)
        res = sharding.sweep_sharded(pts, 3, 8, models.sweep_target(8), tol=1e-12, compute=OracleSweepCompute())
        ap, cv, dg = res.gather()
        q.put((rank, res.start, res.stop, ap, cv, dg))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sweep_sharded_gloo_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2411_09982_b200 import models

    ref = OracleSweepCompute().run(models.sweep_points(3, 3), 3, 8, models.sweep_target(8), 1e-12, None)
    spans = [(g[1], g[2]) for g in got]
    assert spans[0][0] == 0 and spans[-1][1] == 9 and all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    for _, _, _, ap, cv, dg in got:
        np.testing.assert_array_equal(ap, ref[0].numpy())
        np.testing.assert_array_equal(cv, ref[1].numpy().astype(bool))
        np.testing.assert_array_equal(dg, ref[2].numpy())
