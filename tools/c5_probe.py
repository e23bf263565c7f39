"""Config 5 probe: Magnus on the 12-spin Heisenberg chain (dim 4096), order 2,
the first n intervals through evolve_device, with the per-kernel profile.

    python tools/c5_probe.py [n_intervals] [check|nocheck] [repeats]
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import _lib
    from paper_2411_09982_b200 import magnus as mg

    n_int = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    check = len(sys.argv) > 2 and sys.argv[2] == "check"
    ch = eff.heisenberg_chain_hamiltonians(12)
    full = eff.synthetic_transfer_pulse(25.0, 4096 * 8 + 1, seed=7)
    grid = eff.ControlGrid(0.0, 25.0 * n_int / 4096, full.signals[:, : n_int * 8 + 1])
    psi0 = np.zeros(4096, dtype=complex)
    psi0[0] = 1
    d_psi = _lib.to_device(psi0)
    ch.device_operators()
    mg.evolve_device(ch, grid, min(n_int, 8), d_psi, check=check, order=2)  # one full chunk: pool mapped
    torch.cuda.synchronize()
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    for rep in range(reps):
        _lib.profile_read(reset=True)
        _lib.profile_enable(True)
        t0 = time.perf_counter()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        mg.evolve_device(ch, grid, n_int, d_psi, check=check, order=2)
        e.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        _lib.profile_enable(False)
        prof = _lib.profile_read(reset=True)
        ms = s.elapsed_time(e)
        print(f"config 5: {n_int} intervals order 2 check={check}: {ms:.1f} ms (wall {wall * 1e3:.1f}) -> "
              f"{n_int / (ms * 1e-3):.2f} intervals/s", flush=True)
    n = 4096
    for k, (tot, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        extra = ""
        if k.startswith("zgemm"):
            half = "herm" in k
            fl = cnt * n_int * 8.0 * n**3 * (0.5 + 128 / n if half else 1.0)
            extra = f"  executed {fl / (tot * 1e-3) / 1e12:.2f} TFLOP/s"
        print(f"  {k:24s} {tot:10.2f} ms  x{cnt}{extra}", flush=True)


if __name__ == "__main__":
    main()
