"""Print a few rows of the per-tile timeline written by QCH_MAGNUS_STATS=2
(gpurun_out/magnus_tstamp.csv): window landed, prefix known, tile done (us)."""
import numpy as np
d = np.genfromtxt('gpurun_out/magnus_tstamp.csv', delimiter=',', names=True)
w, p, e = d['window_ns']/1e3, d['prefix_ns']/1e3, d['end_ns']/1e3
for t in (0, 16, 31, 100, 147, 148, 200, 295, 296, 390):
    print(f"tile {t:3d}: window {w[t]:7.1f} prefix {p[t]:7.1f} end {e[t]:7.1f}")
print("max end", e.max())
