"""The N > 4 evolve split into many chunks (QCH_EVOLVE_CHUNK caps the
intervals per chunk; read once per process, so each case runs in a child
process): the state hand-over between chunks and the ordered product's
interval offsets, against the order-2 oracle (1e-10) and against the
one-chunk run.  Dims 12 and 64 (one-cluster ordered product) and 400
(cooperative-grid ordered product)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_fro
from oracle import magnus_oracle

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2411_09982_b200 as E
d = np.load(sys.argv[2])
ch = E.ControlledHamiltonian(E.HermitianOperator(d["drift"]), [E.HermitianOperator(c) for c in d["controls"]])
grid = E.ControlGrid(0.0, float(d["t1"]), d["signals"])
out = E.evolve(ch, grid, int(d["m"]), d["psi0"], order=2).amplitudes
np.save(sys.argv[3], out)
"""


def _case(n, k, m, seed):
    rng = np.random.default_rng(seed)

    def herm(scale):
        a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        return scale * (a + a.conj().T) / (2 * np.sqrt(n))

    drift, controls = herm(1.0), np.stack([herm(0.5) for _ in range(k)])
    signals = rng.standard_normal((k, 4 * m + 1))
    psi0 = np.zeros(n, dtype=complex)
    psi0[0] = 1.0
    return drift, controls, signals, psi0


def _run(tmp_path, case, m, t1, chunk):
    drift, controls, signals, psi0 = case
    inp = tmp_path / "in.npz"
    np.savez(inp, drift=drift, controls=controls, signals=signals, psi0=psi0, m=m, t1=t1)
    out = tmp_path / f"out_{chunk}.npy"
    env = dict(os.environ)
    if chunk:
        env["QCH_EVOLVE_CHUNK"] = str(chunk)
    subprocess.run([sys.executable, "-c", CHILD, str(ROOT), str(inp), str(out)], check=True, env=env, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("n,m,chunk", [(12, 23, 5), (64, 17, 4), (400, 5, 2)])
def test_evolve_many_chunks_vs_oracle(tmp_path, n, m, chunk):
    case = _case(n, 2, m, seed=n)
    t1 = 1.5
    drift, controls, signals, psi0 = case
    ref = magnus_oracle.evolve(drift, controls, signals, 0.0, t1, m, psi0, order=2)
    many = _run(tmp_path, case, m, t1, chunk)
    one = _run(tmp_path, case, m, t1, 0)
    assert rel_fro(many, ref) <= 1e-10
    assert rel_fro(many, one) <= 1e-12
