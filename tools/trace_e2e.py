import sys, time, numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2411_09982_b200 as eff
m = 100_000
ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
psi0 = np.array([1, 0, 0], dtype=complex)
sig_p = torch.empty(grid.signals.shape, dtype=torch.float64).pin_memory()
sig_p.numpy()[:] = grid.signals
g2 = eff.ControlGrid(grid.t_start, grid.t_end, sig_p.numpy())
for _ in range(20):
    eff.evolve(ch, g2, m, psi0, order=2, check=False)
torch.cuda.synchronize()
import os
print("---- traced call", file=sys.stderr, flush=True)
eff.evolve(ch, g2, m, psi0, order=2, check=False)
