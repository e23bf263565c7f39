"""Per-rotation latency of ONE sweep chain (the longest of config 4) with each
many-chain driver, alone and among 127 others (the per-GPU shard at N = 8).

    python tools/sweep_chain_probe.py
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import npad as npd

    pts = eff.sweep_points(32, 32)
    tgt = eff.sweep_target(256)
    mats = npd.build_transmon_resonator_batch(pts, 4, 256)
    ap, _ = npd._run_batch_inplace(mats, tgt, 1e-12, None)
    ap = ap.cpu().numpy()
    order = np.argsort(-ap)
    print("longest chains:", [(int(k), int(ap[k])) for k in order[:5]], "mean", ap.mean(), flush=True)
    del mats
    for drv in ("warp", "cta"):
        os.environ["QCH_NPAD_DRIVER"] = drv
        for sel in ([int(order[0])], [int(k) for k in order[:8]], [int(k) for k in order[:128]]):
            best = None
            for _ in range(2):
                m = npd.build_transmon_resonator_batch(pts[sel], 4, 256)
                mx = npd.max_abs_batch(m)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                a2, _ = npd._run_batch_inplace(m, tgt, 1e-12, None, mx)
                e.record()
                torch.cuda.synchronize()
                ms = s.elapsed_time(e)
                best = ms if best is None else min(best, ms)
            print(f"[{drv}] {len(sel)} chains: {best:.3f} ms  -> {best * 1e3 / int(ap[order[0]]):.2f} us/rotation "
                  f"of the longest chain", flush=True)


if __name__ == "__main__":
    main()
