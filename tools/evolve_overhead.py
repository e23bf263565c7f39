"""Host-side cost of the public evolve() call (config 2, pinned signals):
time each Python piece separately.  python tools/evolve_overhead.py"""
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
    g2 = eff.ControlGrid(grid.t_start, grid.t_end, sig_p.numpy())

    def timeit(name, f, n=50):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            f()
        torch.cuda.synchronize()
        print(f"{name:40s} {(time.perf_counter() - t0) / n * 1e6:9.1f} us", flush=True)

    timeit("evolve()", lambda: eff.evolve(ch, g2, m, psi0, order=2, check=False))
    timeit("_evolve_host", lambda: mg._evolve_host(ch, g2, m, psi0, False, 2))
    timeit("_times", lambda: mg._times(g2.t_start, g2.t_end, m))
    timeit("host_empty traj", lambda: _lib.host_empty((m + 1, 3)))
    timeit("np.empty traj", lambda: np.empty((m + 1, 3), complex))
    timeit("host_operators", lambda: ch.host_operators())
    timeit("linspace", lambda: np.linspace(0.0, 100.0, m + 1))


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def profile():
    import cProfile
    import pstats

    import torch

    import paper_2411_09982_b200 as eff

    m = 100_000
    ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
    psi0 = np.array([1, 0, 0], dtype=complex)
    sig_p = torch.empty(grid.signals.shape, dtype=torch.float64).pin_memory()
    sig_p.numpy()[:] = grid.signals
    g2 = eff.ControlGrid(grid.t_start, grid.t_end, sig_p.numpy())
    for _ in range(5):
        eff.evolve(ch, g2, m, psi0, order=2, check=False)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        eff.evolve(ch, g2, m, psi0, order=2, check=False)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)


if __name__ == "__main__" and len(sys.argv) > 1:
    profile()
