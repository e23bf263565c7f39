"""Config 2: the fused kernel's device time (CUDA events around the graph
replay of EvolvePlan, i.e. the bench's `value` step) against the span of its
blocks (QCH_MAGNUS_STATS=2 timeline: first block start .. last block end).
python tools/fused_gap_probe.py"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import magnus as mg

    m = 100_000
    ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
    plan = mg.EvolvePlan(ch, grid, m, np.array([1, 0, 0], dtype=complex), order=2, check=False)
    for _ in range(5):
        plan.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(20):
        e0.record()
        plan.run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"EvolvePlan.run: median {np.median(ts):.1f} us, min {np.min(ts):.1f} us", flush=True)


if __name__ == "__main__":
    main()
