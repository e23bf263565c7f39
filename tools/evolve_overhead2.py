"""Host-side cost of the pieces of the config-2 public evolve() call
(everything but the C call), and the C call alone.
python tools/evolve_overhead2.py"""
import ctypes
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

    def timeit(name, f, n=200):
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            f()
        torch.cuda.synchronize()
        print(f"{name:44s} {(time.perf_counter() - t0) / n * 1e6:9.2f} us", flush=True)

    timeit("host_empty traj (100001x3 c128)", lambda: _lib.host_empty((m + 1, 3), np.complex128))
    timeit("host_empty times", lambda: _lib.host_empty((m + 1,), np.float64))
    timeit("stream_ptr", _lib.stream_ptr)
    timeit("_as_state", lambda: mg._as_state(psi0))
    timeit("_check_intervals", lambda: mg._check_intervals(g2, m))
    timeit("host_operators", lambda: ch.host_operators())
    timeit("ascontiguousarray(signals)", lambda: np.ascontiguousarray(g2.signals))
    timeit("Trajectory(...)", lambda: eff.Trajectory(np.zeros(3), np.zeros((3, 3), complex)))
    timeit("_evolve_host", lambda: mg._evolve_host(ch, g2, m, psi0, False, 2), 50)
    timeit("evolve", lambda: eff.evolve(ch, g2, m, psi0, order=2, check=False), 50)


if __name__ == "__main__":
    main()
