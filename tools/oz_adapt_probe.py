"""Accuracy and speed of the adaptive slice plan (config 5 propagators):
the same 8 intervals on the DMMA engine, the int8 engine with every product
on 8 slices (QCH_OZ_ADAPT=0) and with the adaptive plan; max relative
Frobenius difference per propagator against DMMA, and the chunk time.
python tools/oz_adapt_probe.py"""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import _lib
    from paper_2411_09982_b200 import magnus as mg

    L = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    n = 1 << L
    n_int = 8
    ch = eff.heisenberg_chain_hamiltonians(L)
    full = eff.synthetic_transfer_pulse(25.0, 4096 * 8 + 1, seed=7)
    grid = eff.ControlGrid(0.0, 25.0 * n_int / 4096, full.signals[:, : n_int * 8 + 1])
    psi0 = np.zeros(n, dtype=complex)
    psi0[0] = 1
    d_psi = _lib.to_device(psi0)
    ch.device_operators()
    out = {}
    for name, eng, adapt in (("dmma", 0, "1"), ("int8-8", 1, "0"), ("int8-adapt", 1, "1")):
        os.environ["QCH_OZ_ADAPT"] = adapt
        old = _lib.load().qch_set_herm_gemm(eng)
        props = torch.empty((n_int, n, n), dtype=torch.complex128, device="cuda")
        for _ in range(2):  # warm (allocations, pool growth)
            mg.evolve_device(ch, grid, n_int, d_psi, check=False, order=2, props=props)
        torch.cuda.synchronize()
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            mg.evolve_device(ch, grid, n_int, d_psi, check=False, order=2, props=props)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        _lib.load().qch_set_herm_gemm(old)
        out[name] = props
        print(f"{name:11s} {n_int} intervals {dt * 1e3:8.1f} ms", flush=True)
    ref = out["dmma"]
    for name in ("int8-8", "int8-adapt"):
        d = [float(torch.linalg.norm(out[name][k] - ref[k]) / torch.linalg.norm(ref[k])) for k in range(n_int)]
        print(f"{name:11s} vs dmma: max rel fro {max(d):.3e}", flush=True)
    d = [float(torch.linalg.norm(out["int8-adapt"][k] - out["int8-8"][k]) / torch.linalg.norm(ref[k]))
         for k in range(n_int)]
    print(f"adapt vs int8-8: max rel fro {max(d):.3e}", flush=True)


if __name__ == "__main__":
    main()
