"""Config-4 sweep scaling model measured on ONE GPU: the sweep has no
exchange, so an N-GPU run is N independent shards and its makespan is the
slowest shard.  For N = 1, 2, 4, 8 every shard (sharding.shard_bounds of the
1024 points) is solved alone on this GPU with each many-chain driver, timed
with CUDA events; prints per-shard ms, the predicted makespan and speed-up.

    python tools/sweep_scale_probe.py [drivers=warp,cta,auto]
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import npad as npd
    from paper_2411_09982_b200.sharding import shard_bounds

    drivers = (sys.argv[1] if len(sys.argv) > 1 else "warp,cta,auto").split(",")
    pts = eff.sweep_points(32, 32)
    tgt = eff.sweep_target(256)
    out = {}
    for drv in drivers:
        if drv == "auto":
            os.environ.pop("QCH_NPAD_DRIVER", None)
        else:
            os.environ["QCH_NPAD_DRIVER"] = drv
        res = {}
        for world in (1, 2, 4, 8):
            shard_ms = []
            for r in range(world):
                a, b = shard_bounds(len(pts), world, r)
                best = None
                for _ in range(2):
                    mats = npd.build_transmon_resonator_batch(pts[a:b], 4, 256)
                    mx = npd.max_abs_batch(mats)
                    torch.cuda.synchronize()
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    ap, cv = npd._run_batch_inplace(mats, tgt, 1e-12, None, mx)
                    e.record()
                    torch.cuda.synchronize()
                    ms = s.elapsed_time(e)
                    best = ms if best is None else min(best, ms)
                    rot = int(ap.sum().item())
                    del mats
                shard_ms.append(best)
            res[world] = {"shard_ms": shard_ms, "makespan_ms": max(shard_ms)}
            print(f"[{drv}] N={world}: makespan {max(shard_ms):.2f} ms  shards {[round(x, 2) for x in shard_ms]}",
                  flush=True)
        base = res[1]["makespan_ms"]
        for w in res:
            res[w]["speedup"] = base / res[w]["makespan_ms"]
        out[drv] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()
