"""Phase counters of the fused kernel inside the host-buffer evolve (zero-copy
I/O): QCH_MAGNUS_STATS=1 python tools/host_stats.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2411_09982_b200 as eff

    m = 100_000
    ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
    sig_p = torch.empty(grid.signals.shape, dtype=torch.float64).pin_memory()
    sig_p.numpy()[:] = grid.signals
    g2 = eff.ControlGrid(grid.t_start, grid.t_end, sig_p.numpy())
    for _ in range(3):
        eff.evolve(ch, g2, m, np.array([1, 0, 0], dtype=complex), order=2, check=False)


if __name__ == "__main__":
    main()
