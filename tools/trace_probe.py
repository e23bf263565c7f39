"""CUPTI timeline (torch.profiler) of one device evolve at spin-chain length
L (argv[1], default 8; argv[2] intervals; argv[3] = c5: config 5's pulse): kernels, runtime API calls that block or allocate,
and the idle gaps between kernels.  python tools/trace_probe.py 8"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import _lib
    from paper_2411_09982_b200 import magnus as mg

    L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    m = int(sys.argv[2]) if len(sys.argv) > 2 else {6: 4096, 8: 2048, 10: 256}.get(L, 512)
    n = 1 << L
    ch = eff.heisenberg_chain_hamiltonians(L)
    if len(sys.argv) > 3 and sys.argv[3] == "c5":  # config 5's pulse: 25 time units over 4096 intervals
        full = eff.synthetic_transfer_pulse(25.0, 4096 * 8 + 1, seed=7)
        grid = eff.ControlGrid(0.0, 25.0 * m / 4096, full.signals[:, : m * 8 + 1])
    else:
        pulse = eff.synthetic_transfer_pulse(25.0, m * 8 + 1, seed=7)
        grid = eff.ControlGrid(0.0, 25.0, pulse.signals)
    psi0 = np.zeros(n, dtype=complex)
    psi0[0] = 1
    d_psi = _lib.to_device(psi0)
    ch.device_operators()
    for _ in range(2):
        mg.evolve_device(ch, grid, m, d_psi, check=False, order=2)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        mg.evolve_device(ch, grid, m, d_psi, check=False, order=2)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    last = t0
    print(f"L={L} N={n} M={m}: {len(evs)} device events over {(evs[-1].time_range.end - t0) / 1e3:.2f} ms")
    gaps = 0.0
    for e in evs:
        g = e.time_range.start - last
        if g > 20:
            gaps += g
        if len(evs) <= 60:
            print(f"  +{(e.time_range.start - t0) / 1e3:8.3f} ms  gap {g / 1e3:7.3f}  "
                  f"{e.time_range.elapsed_us() / 1e3:8.3f} ms  {e.name[:70]}")
        last = max(last, e.time_range.end)
    print(f"  idle gaps > 20 us: {gaps / 1e3:.2f} ms")
    per = {}
    for e in evs:
        a = per.setdefault(e.name[:60], [0, 0.0])
        a[0] += 1
        a[1] += e.time_range.elapsed_us()
    for k, (c, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"  {us / 1e3:10.3f} ms x{c:4d}  {k}")
    cpu = [e for e in prof.events() if e.device_type.name == "CPU" and e.name.startswith("cuda")]
    agg = {}
    for e in cpu:
        a = agg.setdefault(e.name, [0, 0.0])
        a[0] += 1
        a[1] += e.time_range.elapsed_us()
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"  {k:40s} x{c:5d} {us / 1e3:8.3f} ms")


if __name__ == "__main__":
    main()
