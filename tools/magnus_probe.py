"""Where does the config-2 e2e time go?  Times each piece of the public
evolve() call on the GPU box (perf_counter around synchronised pieces) and
the fused kernel alone (CUDA events).  python tools/magnus_probe.py"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import _lib
    from paper_2411_09982_b200 import magnus as mg

    m = 100_000
    ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
    psi0 = np.array([1, 0, 0], dtype=complex)
    sig_p = torch.empty(grid.signals.shape, dtype=torch.float64).pin_memory()
    sig_p.numpy()[:] = grid.signals
    ops = [ch.drift.data] + [c.data for c in ch.controls]

    def timeit(name, f, n=20):
        f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            f()
        torch.cuda.synchronize()
        print(f"{name:40s} {(time.perf_counter() - t0) / n * 1e6:10.1f} us")

    timeit("ControlGrid(pinned signals)", lambda: eff.ControlGrid(grid.t_start, grid.t_end, sig_p.numpy()))
    timeit("3x HermitianOperator", lambda: [eff.HermitianOperator(o, validate=False) for o in ops])
    g2 = eff.ControlGrid(grid.t_start, grid.t_end, sig_p.numpy())
    timeit("evolve (host path, pinned)", lambda: eff.evolve(ch, g2, m, psi0, order=2, check=False))
    timeit("evolve (host path, pageable)", lambda: eff.evolve(ch, grid, m, psi0, order=2, check=False))
    import os
    for env in ({}, {"QCH_NOMAP_SIG": "1"}, {"QCH_NOMAP_TRAJ": "1"}, {"QCH_NOMAP_SIG": "1", "QCH_NOMAP_TRAJ": "1"},
                {"QCH_STREAM_BPS": "2"}, {"QCH_STREAM_BPS": "3"}, {"QCH_STREAM_BPS": "0"}):
        os.environ.update(env)
        timeit(f"evolve pinned {sorted(env)}", lambda: eff.evolve(ch, g2, m, psi0, order=2, check=False))
        for k in env:
            del os.environ[k]
    os.environ["QCH_TRACE"] = "1"
    for _ in range(3):
        t0 = time.perf_counter()
        eff.evolve(ch, g2, m, psi0, order=2, check=False)
        print(f"evolve wall {(time.perf_counter() - t0) * 1e6:.1f} us", file=sys.stderr, flush=True)
    del os.environ["QCH_TRACE"]
    import cProfile
    import pstats

    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        eff.evolve(ch, g2, m, psi0, order=2, check=False)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
    timeit("host_empty traj", lambda: _lib.host_empty((m + 1, 3)))
    timeit("_times", lambda: mg._times(0.0, 100.0, m))
    d_psi = _lib.to_device(psi0)
    timeit("evolve_device (sync)", lambda: mg.evolve_device(ch, grid, m, d_psi, check=False, order=2))
    # raw transfers
    d = torch.empty(grid.signals.shape, dtype=torch.float64, device="cuda")
    timeit("H2D 6.4 MB pinned", lambda: d.copy_(sig_p, non_blocking=True))
    tr = torch.empty((m + 1, 3), dtype=torch.complex128, device="cuda")
    hp = torch.empty((m + 1, 3), dtype=torch.complex128).pin_memory()
    timeit("D2H 4.8 MB pinned", lambda: hp.copy_(tr, non_blocking=True))
    # kernel alone
    _lib.profile_read(reset=True)
    _lib.profile_enable(True)
    for _ in range(5):
        mg.evolve_device(ch, grid, m, d_psi, check=False, order=2)
    _lib.profile_enable(False)
    for k, (ms, n) in _lib.profile_read(reset=True).items():
        print(f"kernel {k:32s} {ms / n * 1e3:10.1f} us x{n}")
    for order in (1, 2):
        _lib.profile_enable(True)
        for _ in range(5):
            mg.evolve_device(ch, grid, m, d_psi, check=True, order=order)
        _lib.profile_enable(False)
        for k, (ms, n) in _lib.profile_read(reset=True).items():
            print(f"kernel order={order} check {k:24s} {ms / n * 1e3:10.1f} us x{n}")


if __name__ == "__main__":
    main()
