"""Config 2 (headline) device-resident step: EvolvePlan.run() timed with
CUDA events, with and without an L2 flush before each step.  Under ncu
(--metrics gpu__time_duration.sum) it gives the kernel's own duration.
python tools/plan_probe.py [reps]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import magnus as mg

    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    m = 100_000
    ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
    psi0 = np.array([1, 0, 0], dtype=complex)
    plan = mg.EvolvePlan(ch, grid, m, psi0, order=2, check=False)
    for _ in range(5):
        plan.run()
    torch.cuda.synchronize()
    junk = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for flush in (False, True):
        ts = []
        for _ in range(reps):
            if flush:
                junk.fill_(1.0)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            plan.run()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        print(f"flush={flush}: median {np.median(ts):.1f} us, min {np.min(ts):.1f} us", flush=True)


if __name__ == "__main__":
    main()
