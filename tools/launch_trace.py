"""Launch-call timing of the fused Magnus kernel (device path, then host-buffer
path): QCH_TRACE=1 python tools/launch_trace.py"""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2411_09982_b200 as eff
from paper_2411_09982_b200 import magnus as mg
m = 100_000
ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
d = torch.tensor(np.array([1, 0, 0], dtype=complex), device="cuda")
for _ in range(4):
    mg.evolve_device(ch, grid, m, d, check=False, order=2)
sig_p = torch.empty(grid.signals.shape, dtype=torch.float64).pin_memory(); sig_p.numpy()[:] = grid.signals
g2 = eff.ControlGrid(grid.t_start, grid.t_end, sig_p.numpy())
for _ in range(4):
    eff.evolve(ch, g2, m, np.array([1, 0, 0], dtype=complex), order=2, check=False)
