"""NPAD parameter sweep across devices / ranks (config 4 host paths) on ONE
GPU: npad_run_batch(devices=[0, 0]) (two host threads, one block each),
non-bitwise-Hermitian operators routed to the single-chain driver inside a
batch, the batched max_abs, and sharding.sweep_sharded in a world-1 NCCL
group.  Per-point results must equal npad_run / the oracle exactly."""
import os
import socket

import numpy as np
import pytest

from conftest import rel_fro
from oracle import npad_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


def _pts(E, k=6):
    return E.sweep_points(3, 2)[:k]


def _h(E, pt, n_q=3, n_r=10):
    wq, al, wr, g = pt
    return E.transmon_resonator_hamiltonian(n_q, n_r, omega_q=wq, alpha=al, omega_r=wr, g=g).data


def test_batch_devices_split_and_nonhermitian_routing(E):
    pts = _pts(E)
    tgt = E.sweep_target(10)
    hs = [_h(E, p) for p in pts]
    # point 2: Hermitian only to rounding (not bitwise) -> single-chain driver
    rng = np.random.default_rng(0)
    pert = 1e-15 * (rng.standard_normal(hs[2].shape) + 1j * rng.standard_normal(hs[2].shape))
    hs[2] = hs[2] + np.triu(pert, 1)
    refs = [npad_oracle.run_incremental(h, tgt, tol=1e-12) for h in hs]
    for devices in (None, [0, 0], [0, 0, 0]):
        res = E.npad_run_batch([E.HermitianOperator(h, validate=False) for h in hs], tgt, tol=1e-12,
                               devices=devices)
        assert len(res.parts) == (1 if devices is None else len(devices))
        for k, r in enumerate(refs):
            assert int(res.applied[k]) == r["applied"] and bool(res.converged[k]) == r["converged"]
            assert rel_fro(res.operator(k).data, r["h"]) <= 1e-10
        np.testing.assert_allclose(res.diagonals(), np.stack([np.real(np.diag(r["h"])) for r in refs]), rtol=0,
                                   atol=1e-9)


def test_max_abs_batch_matches_single(E):
    import torch

    from paper_2411_09982_b200 import npad

    mats = npad.build_transmon_resonator_batch(_pts(E), 3, 10)
    got = npad.max_abs_batch(mats).cpu().numpy()
    for k in range(mats.shape[0]):
        assert got[k] == E.HermitianOperator(mats[k].cpu().numpy()).max_abs()
    assert isinstance(mats, torch.Tensor)
    # the builder's own max (formed while writing) and its matrices equal the host builder
    pts = E.sweep_points(4, 4)
    m2, mx = npad.build_transmon_resonator_batch(pts, 4, 64, with_max_abs=True)
    for k in (0, 7, 15):
        wq, al, wr, g = pts[k]
        host = E.transmon_resonator_hamiltonian(4, 64, omega_q=wq, alpha=al, omega_r=wr, g=g).data
        np.testing.assert_array_equal(m2[k].cpu().numpy(), host)
        assert float(mx[k].item()) == float(np.max(np.abs(host)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sweep_sharded_world1_nccl(E):
    import torch.distributed as dist

    from paper_2411_09982_b200 import sharding

    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        pts = _pts(E)
        tgt = E.sweep_target(10)
        res = sharding.sweep_sharded(pts, 3, 10, tgt, tol=1e-12)
        ap, cv, dg = res.gather()
        assert (res.start, res.stop) == (0, len(pts))
        for k, p in enumerate(pts):
            r = npad_oracle.run_incremental(_h(E, p), tgt, tol=1e-12)
            assert ap[k] == r["applied"] and cv[k] == r["converged"]
            assert rel_fro(dg[k], np.real(np.diag(r["h"]))) <= 1e-10
    finally:
        dist.destroy_process_group()
