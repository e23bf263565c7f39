"""The N > 4 Magnus relay (sharding.evolve_relay) on ONE GPU: the device
compute (qch_magnus_propagators_c128 on a chunk's signal window +
qch_magnus_chain_c128 from the relayed state) driven in round-robin chunk
order as W ranks would, the world-1 NCCL driver with the gather, and config 5
at dim 4096 against the order-2 oracle golden.  Bar: 1e-10 relative."""
import os
import socket
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_fro
from oracle import magnus_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


def _spin(E, L, m, sub=4, t=2.0, seed=7):
    ch = E.heisenberg_chain_hamiltonians(L)
    grid = E.synthetic_transfer_pulse(t, m * sub + 1, seed=seed)
    psi0 = np.zeros(1 << L, dtype=complex)
    psi0[0] = 1.0
    return ch, grid, psi0


@pytest.mark.parametrize("L,m,chunk,world", [(6, 24, 3, 4), (6, 10, 4, 2), (8, 6, 1, 3)])
def test_relay_emulated_ranks_vs_oracle(E, L, m, chunk, world):
    from paper_2411_09982_b200 import sharding

    ch, grid, psi0 = _spin(E, L, m)
    ref = magnus_oracle.evolve(ch.drift.to_dense(), np.stack([c.to_dense() for c in ch.controls]), grid.signals,
                               grid.t_start, grid.t_end, m, psi0, order=2)
    sub = (grid.samples - 1) // m
    dt_int = (grid.t_end - grid.t_start) / m
    ranks = [sharding.DeviceRelayCompute() for _ in range(world)]
    for c in ranks:
        c.setup(ch, 2)
    psi = ranks[0].to_tensor(psi0)
    rows_all = [psi.cpu().numpy()[None]]
    for k in range(-(-m // chunk)):
        comp = ranks[k % world]
        a, b = k * chunk, min(m, (k + 1) * chunk)
        u, err = comp.propagators(ch, grid.signals[:, a * sub: b * sub + 1], grid.dt, dt_int, b - a, 2, True)
        assert err is None
        rows, err = comp.chain(u, b - a, psi.clone())
        assert err is None
        rows_all.append(rows.cpu().numpy())
        psi = rows[-1]
    got = np.concatenate(rows_all)
    assert rel_fro(got, ref) <= 1e-10
    assert rel_fro(got, E.evolve(ch, grid, m, psi0, order=2).amplitudes) <= 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_relay_driver_world1_nccl_and_gather(E):
    import torch.distributed as dist

    from paper_2411_09982_b200 import sharding

    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        m = 8
        ch, grid, psi0 = _spin(E, 8, m)
        ref = E.evolve(ch, grid, m, psi0, order=2).amplitudes
        plan = sharding.RelayEvolvePlan(ch, grid, m, psi0, order=2, check=True, chunk=3)
        for _ in range(2):
            res = plan.run()
        assert [(a, b) for a, b, _ in res.chunks] == [(0, 3), (3, 6), (6, 8)]
        assert rel_fro(res.gather().cpu().numpy(), ref) <= 1e-12
    finally:
        dist.destroy_process_group()


def test_relay_config5_vs_order2_golden(E):
    # BASELINE config 5 (dim 4096, order 2) through the relay path, one
    # interval per chunk
    from paper_2411_09982_b200 import sharding

    g = np.load(Path(__file__).parent / "golden" / "magnus_config5_mid_order2_oracle.npz")
    ch = E.heisenberg_chain_hamiltonians(12)
    t0, t1 = (float(x) for x in g["t"])
    grid = E.ControlGrid(t0, t1, g["signals"])
    res = sharding.evolve_relay(ch, grid, 2, g["traj"][0], order=2, check=True, chunk=1)
    assert rel_fro(res.gather().cpu().numpy(), g["traj"]) <= 1e-10
