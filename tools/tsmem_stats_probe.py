"""Phase counters of the shared-memory sweep driver on the longest config-4
chain (QCH_NPAD_STATS=1): python tools/tsmem_stats_probe.py"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["QCH_NPAD_STATS"] = "1"
os.environ["QCH_NPAD_DRIVER"] = "tsmem"


def main():
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import npad as npd

    pts = eff.sweep_points(32, 32)[[1013, 500, 20]]
    for _ in range(2):
        m = npd.build_transmon_resonator_batch(pts, 4, 256)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ap, _ = npd._run_batch_inplace(m, eff.sweep_target(256), 1e-12, None)
        e.record()
        torch.cuda.synchronize()
        print("ms", s.elapsed_time(e), "applied", ap.cpu().numpy(), flush=True)


if __name__ == "__main__":
    main()
