"""Per-tile timeline of the host-buffer evolve (config 2) under each I/O
mode: when each tile's signal window landed, when its prefix arrived and
when its trajectory was written (globaltimer, QCH_MAGNUS_STATS=2).
python tools/e2e_timeline.py 2>/dev/null   (wall times include the stats overhead)"""
import os
import shutil
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    os.environ["QCH_MAGNUS_STATS"] = "2"  # read once by the library: set before the first launch
    import torch

    import paper_2411_09982_b200 as eff

    m = 100_000
    ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
    psi0 = np.array([1, 0, 0], dtype=complex)
    sig_p = torch.empty(grid.signals.shape, dtype=torch.float64).pin_memory()
    sig_p.numpy()[:] = grid.signals
    g2 = eff.ControlGrid(grid.t_start, grid.t_end, sig_p.numpy())
    Path("gpurun_out").mkdir(exist_ok=True)
    for name, env in (("map", {}), ("stream", {"QCH_SIG_MODE": "stream"}), ("copy", {"QCH_SIG_MODE": "copy"})):
        os.environ.update(env)
        for _ in range(3):
            eff.evolve(ch, g2, m, psi0, order=2, check=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            eff.evolve(ch, g2, m, psi0, order=2, check=False)
        wall = (time.perf_counter() - t0) / 10 * 1e6
        eff.evolve(ch, g2, m, psi0, order=2, check=False)
        for k in env:
            del os.environ[k]
        src = Path("gpurun_out/magnus_tstamp.csv")
        if src.exists():
            shutil.copy(src, f"gpurun_out/tstamp_{name}.csv")
            a = np.loadtxt(src, delimiter=",", skiprows=1)
            w, p, e = a[:, 2] / 1e3, a[:, 3] / 1e3, a[:, 4] / 1e3
            q = lambda x: " ".join(f"{v:6.1f}" for v in np.percentile(x, [0, 25, 50, 75, 100]))  # noqa: E731
            print(f"{name:7s} wall {wall:7.1f} us | window us {q(w)} | prefix us {q(p)} | end us {q(e)}", flush=True)
            # tiles in order: is the prefix front monotone?
            idx = np.argsort(a[:, 0])
            print("   tile-order prefix (every 40th):", " ".join(f"{v:.0f}" for v in p[idx][::40]), flush=True)
            print("   tile-order window (every 40th):", " ".join(f"{v:.0f}" for v in w[idx][::40]), flush=True)


if __name__ == "__main__":
    main()
