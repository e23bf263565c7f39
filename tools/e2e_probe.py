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
    # transfer floor on this box: H2D of the signals || D2H of a trajectory
    d_sig = torch.empty(grid.signals.shape, dtype=torch.float64, device="cuda")
    d_tr = torch.empty((m + 1, 3), dtype=torch.complex128, device="cuda")
    h_tr = torch.empty((m + 1, 3), dtype=torch.complex128).pin_memory()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, fn in (("H2D 6.4 MB", lambda: d_sig.copy_(sig_p, non_blocking=True)),
                     ("D2H 4.8 MB", lambda: h_tr.copy_(d_tr, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        print(f"{name:60s} wall {(time.perf_counter() - t0) / 20 * 1e6:8.1f} us")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        with torch.cuda.stream(s1):
            d_sig.copy_(sig_p, non_blocking=True)
        with torch.cuda.stream(s2):
            h_tr.copy_(d_tr, non_blocking=True)
        torch.cuda.synchronize()
    print(f"{'H2D || D2H':60s} wall {(time.perf_counter() - t0) / 20 * 1e6:8.1f} us")
    for env in ({}, {"QCH_STREAM_BPS": "2"}, {"QCH_STREAM_BPS": "3"}, {"QCH_SIG_MODE": "stream"},
                {"QCH_SIG_MODE": "copy"}, {"QCH_NOMAP_TRAJ": "1"},
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
    os.environ["QCH_MAGNUS_STATS"] = "1"
    for _ in range(2):
        eff.evolve(ch, g2, m, psi0, order=2, check=False)


if __name__ == "__main__":
    main()
