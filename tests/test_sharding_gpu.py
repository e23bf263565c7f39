"""Multi-GPU Magnus sharding on ONE GPU: the per-rank device compute
(qch_magnus_shard_prepare/finish: fused kernel in prefix mode + prefix
mat-vec pass) emulating several ranks in sequence, and the plan / driver with
a world-size-1 NCCL group.  Bar: 1e-10 relative (north star)."""
import os
import socket

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
    return magnus_oracle.evolve(ch.drift.data, np.stack([c.data for c in ch.controls]), grid.signals, grid.t_start,
                                grid.t_end, m, psi0, order=order)


@pytest.mark.parametrize("world,m", [(1, 1000), (3, 20_000), (8, 100_003 - 3), (5, 17)])
def test_emulated_ranks_match_oracle(E, world, m):
    import torch

    from paper_2411_09982_b200 import sharding

    ch, grid = E.driven_transmon(3, intervals=m, sub=4, t_final=100.0 * m / 100_000 + 1.0)
    psi0 = np.array([1, 0, 0], dtype=complex)
    comp = sharding.DeviceMagnusCompute()
    sub = (grid.samples - 1) // m
    dt_int = (grid.t_end - grid.t_start) / m
    parts = []
    for r in range(world):
        a, b = sharding.shard_bounds(m, world, r)
        blk, handle = comp.prepare(ch, grid.signals[:, a * sub: b * sub + 1], grid.dt, dt_int, b - a, 2, True)
        parts.append((a, b, blk, handle))
    blocks = torch.stack([p[2] for p in parts]).contiguous()
    ref = _oracle(ch, grid, m, psi0, 2)
    for r, (a, b, _blk, handle) in enumerate(parts):
        ps = comp.apply_prefix(blocks, r, comp.to_tensor(psi0))
        traj = comp.finish(handle, ps).cpu().numpy()
        assert traj.shape == (b - a + 1, 3)
        assert rel_fro(traj, ref[a:b + 1]) <= 1e-10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_plan_and_driver_world1_nccl(E):
    import torch.distributed as dist

    from paper_2411_09982_b200 import sharding

    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1)
    m = 100_000
    ch, grid = E.driven_transmon(3, intervals=m, sub=4)
    psi0 = np.array([1, 0, 0], dtype=complex)
    ref = _oracle(ch, grid, m, psi0, 2)
    plan = sharding.ShardedEvolvePlan(ch, grid, m, psi0, order=2, check=True)
    for _ in range(3):
        out = plan.run()
    plan.check()
    assert rel_fro(out.cpu().numpy(), ref) <= 1e-10
    res = sharding.evolve_sharded(ch, grid, m, psi0, order=2, check=True)
    assert res.start == 0 and res.stop == m
    assert rel_fro(res.trajectory.cpu().numpy(), ref) <= 1e-10
    dist.destroy_process_group()
