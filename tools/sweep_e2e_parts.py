"""Config 4 end to end, piece by piece: device build of the 1024 points,
the batched solve (row-state init + drivers), diagonals to the host.
python tools/sweep_e2e_parts.py"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import _lib
    from paper_2411_09982_b200 import npad as npd

    n_q, n_r = 4, 256
    pts = eff.sweep_points(32, 32)
    tgt = eff.sweep_target(n_r)
    for rep in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        _lib.profile_read(reset=True)
        _lib.profile_enable(True)
        t0 = time.perf_counter()
        ev[0].record()
        mats, mx = npd.build_transmon_resonator_batch(pts, n_q, n_r, with_max_abs=True)
        ev[1].record()
        applied, conv = npd._run_batch_inplace(mats, tgt, 1e-12, None, mx)
        ev[2].record()
        res = npd.BatchResult([(0, mats)], _lib.to_host(applied), _lib.to_host(conv).astype(bool))
        dg = res.diagonals()
        ev[3].record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        _lib.profile_enable(False)
        prof = _lib.profile_read(reset=True)
        print(f"rep {rep}: build {ev[0].elapsed_time(ev[1]):.2f} ms, solve {ev[1].elapsed_time(ev[2]):.2f} ms, "
              f"diagonals {ev[2].elapsed_time(ev[3]):.2f} ms, wall {wall:.2f} ms | "
              + ", ".join(f"{k} {v[0]:.2f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])), flush=True)
        del mats, mx, res


if __name__ == "__main__":
    main()
