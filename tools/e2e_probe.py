"""Kernel-side view of the host-buffer evolve (config 2): fused-kernel time
(CUDA events) and wall time of evolve() for zero-copy vs staged I/O and
streaming grid sizes.  python tools/e2e_probe.py"""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import _lib

    m = 100_000
    ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
    psi0 = np.array([1, 0, 0], dtype=complex)
    sig_p = torch.empty(grid.signals.shape, dtype=torch.float64).pin_memory()
    sig_p.numpy()[:] = grid.signals
    g2 = eff.ControlGrid(grid.t_start, grid.t_end, sig_p.numpy())
    for env in ({}, {"QCH_SIG_CHUNKS": "4"}, {"QCH_SIG_CHUNKS": "16"}, {"QCH_SIG_CHUNKS": "32"},
                {"QCH_SIG_MODE": "map"}, {"QCH_SIG_MODE": "copy"}, {"QCH_NOMAP_TRAJ": "1"},
                {"QCH_SIG_MODE": "copy", "QCH_NOMAP_TRAJ": "1"}):
        os.environ.update(env)
        for _ in range(3):
            eff.evolve(ch, g2, m, psi0, order=2, check=False)
        torch.cuda.synchronize()
        _lib.profile_read(reset=True)
        _lib.profile_enable(True)
        t0 = time.perf_counter()
        n = 20
        for _ in range(n):
            eff.evolve(ch, g2, m, psi0, order=2, check=False)
        wall = (time.perf_counter() - t0) / n * 1e6
        _lib.profile_enable(False)
        prof = _lib.profile_read(reset=True)
        k = prof.get("magnus_fused_kernel", (0, 1))
        print(f"{str(sorted(env.items())):60s} wall {wall:8.1f} us   kernel {k[0] / k[1] * 1e3:8.1f} us")
        for key in env:
            del os.environ[key]


if __name__ == "__main__":
    main()
