"""Per-rank work of the config-2 interval sharding (N <= 4) on ONE GPU: the
ShardedEvolvePlan step (pass 1 in prefix mode, the block all-gather in an
NCCL world of 1, apply-prefix, pass 2) vs the single-GPU EvolvePlan step,
both 10^5 intervals, CUDA events, L2 flushed.

    python tools/shard_probe.py
"""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import magnus as mg
    from paper_2411_09982_b200 import sharding

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
    s.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    m = 100_000
    ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
    psi0 = np.array([1, 0, 0], dtype=complex)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for name, plan in (("EvolvePlan", mg.EvolvePlan(ch, grid, m, psi0, order=2, check=False)),
                       ("ShardedEvolvePlan", sharding.ShardedEvolvePlan(ch, grid, m, psi0, order=2, check=False))):
        for _ in range(5):
            plan.run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            plan.run()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        print(f"{name}: median {ts[len(ts) // 2] * 1e3:.1f} us/step, min {ts[0] * 1e3:.1f}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
