"""mid-size dense propagation (spin chains L = 6..10,
N = 64..1024) — batched expm and evolve throughput against the DMMA peak.
python tools/midsize_probe.py"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import _lib
    from paper_2411_09982_b200 import expm as ex
    from paper_2411_09982_b200 import magnus as mg

    for L, m in ((6, 4096), (8, 2048), (10, 256)):
        n = 1 << L
        ch = eff.heisenberg_chain_hamiltonians(L)
        pulse = eff.synthetic_transfer_pulse(25.0, m * 8 + 1, seed=7)
        grid = eff.ControlGrid(0.0, 25.0, pulse.signals)
        psi0 = np.zeros(n, dtype=complex)
        psi0[0] = 1
        d_psi = _lib.to_device(psi0)
        ch.device_operators()
        for check in (False, True):
            mg.evolve_device(ch, grid, m, d_psi, check=check, order=2)
            torch.cuda.synchronize()
            _lib.profile_read(reset=True)
            _lib.profile_enable(True)
            t0 = time.perf_counter()
            reps = 3
            for _ in range(reps):
                mg.evolve_device(ch, grid, m, d_psi, check=check, order=2)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / reps
            _lib.profile_enable(False)
            prof = _lib.profile_read(reset=True)
            g_ms = sum(v[0] for k, v in prof.items() if k.startswith("zgemm")) / reps
            g_cnt = sum(v[1] for k, v in prof.items() if k.startswith("zgemm")) / reps
            tot_ms = sum(v[0] for v in prof.values()) / reps
            print(f"L={L:2d} N={n:5d} M={m:5d} check={check!s:5s}: {m / dt:10.1f} intervals/s "
                  f"({dt * 1e3:8.2f} ms), kernels {tot_ms:8.2f} ms, GEMM {g_ms:8.2f} ms in {g_cnt:.0f} launches",
                  flush=True)
            if not check:
                top = sorted(prof.items(), key=lambda kv: -kv[1][0])[:6]
                print("    " + ", ".join(f"{k} {v[0] / reps:.2f} ms x{v[1] / reps:.0f}" for k, v in top), flush=True)
        # batched expm alone
        b = min(m, 512)
        h = torch.randn((b, n, n), dtype=torch.complex128, device="cuda") * (0.2 / n ** 0.5)
        h = 0.5 * (h + h.transpose(1, 2).conj())
        ex.expm_device(h)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            ex.expm_device(h)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 3
        print(f"    expm_device batch {b} x N={n}: {b / dt:10.1f} matrices/s ({dt * 1e3:.2f} ms)", flush=True)


if __name__ == "__main__":
    main()
