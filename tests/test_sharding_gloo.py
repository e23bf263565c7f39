"""Multi-process (world_size 2, gloo, CPU) test of the sharding host logic:
interval partition, the all-gather of block products and the prefix order.
The per-rank compute is the CPU oracle injected in place of the GPU kernels;
the distributed result must equal the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import expm_oracle, magnus_oracle


class OracleCompute:
    def prepare(self, ch, sig, dt, dt_int, m_local, order, check):
        steps = sig.shape[1] - 1
        t0, t1 = 0.0, dt * steps
        hb = magnus_oracle.effective_hamiltonians(ch.drift.data, np.stack([c.data for c in ch.controls]), sig, t0, t1,
                                                  m_local, order)
        us = [expm_oracle.expm_minus_i(h) for h in hb]
        block = np.eye(ch.dim, dtype=complex)
        for u in us:
            block = u @ block
        return torch.from_numpy(block), us

    def apply_prefix(self, blocks, rank, psi0):
        v = psi0.numpy().copy()
        for b in range(rank):
            v = blocks[b].numpy() @ v
        return torch.from_numpy(v)

    def finish(self, us, psi_start):
        v = psi_start.numpy()
        out = [v]
        for u in us:
            v = u @ v
            out.append(v)
        return torch.from_numpy(np.stack(out))

    def to_tensor(self, psi0):
        return torch.from_numpy(np.asarray(psi0, dtype=complex))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_09982_b200 import models, sharding

        ch, grid = models.driven_transmon(3, intervals=m, sub=4, t_final=10.0, amplitude=0.3)
        res = sharding.evolve_sharded(ch, grid, m, np.array([1, 0, 0], dtype=complex), order=2,
                                      compute=OracleCompute())
        q.put((rank, res.start, res.stop, res.trajectory.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(2, 40), (2, 9), (3, 10)])
def test_evolve_sharded_gloo_matches_single_process(world, m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2411_09982_b200 import models

    ch, grid = models.driven_transmon(3, intervals=m, sub=4, t_final=10.0, amplitude=0.3)
    ref = magnus_oracle.evolve(ch.drift.data, np.stack([c.data for c in ch.controls]), grid.signals, grid.t_start,
                               grid.t_end, m, np.array([1, 0, 0], dtype=complex), order=2)
    got.sort()
    assert got[0][1] == 0 and got[-1][2] == m
    for rank, start, stop, traj in got:
        assert traj.shape == (stop - start + 1, 3)
        np.testing.assert_allclose(traj, ref[start:stop + 1], rtol=0, atol=1e-12)
    # contiguous, non-overlapping blocks
    for a, b in zip(got, got[1:]):
        assert a[2] == b[1]


def test_shard_bounds_cover_exactly():
    from paper_2411_09982_b200.sharding import shard_bounds

    for total in (1, 7, 8, 100000, 1024):
        for world in (1, 2, 3, 8):
            if total < world:
                continue
            spans = [shard_bounds(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
