"""DMMA zgemm probe: TMA kernel vs the cp.async kernel vs cuBLAS (torch), and
the Hermitian half-GEMM, at N = 4096 (and a batch of 1024^2).  Prints
TFLOP/s credited at 8 N^3 per complex GEMM (Hermitian: the full 8 N^3 it
replaces, and the executed half).

    python tools/zgemm_probe.py [n] [reps]
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def run(n: int, reps: int, label: str):
    import torch

    from paper_2411_09982_b200 import _lib

    lib = _lib.load()
    a = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    h = (a + a.mH) * 0.5
    b = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    c = torch.empty_like(a)
    sp = _lib.stream_ptr()

    def t(fn):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    fl = 8.0 * n**3
    ms = t(lambda: lib.qch_zgemm_batched(_lib.dptr(a), _lib.dptr(b), _lib.dptr(c), n, n, n, 1, n * n, n * n, n * n, sp))
    ref = a @ b
    err = float((c - ref).abs().max() / ref.abs().max())
    print(f"[{label}] zgemm {n}: {ms:.3f} ms  {fl / ms / 1e9:.2f} TFLOP/s  maxrel {err:.1e}", flush=True)
    if label == "tma":
        h2 = h @ h
        ms_h = t(lambda: lib.qch_zgemm_herm_batched(_lib.dptr(h2), _lib.dptr(h), _lib.dptr(c), n, 1, sp))
        ref = h2 @ h
        err = float((c - ref).abs().max() / ref.abs().max())
        print(f"[{label}] herm {n}: {ms_h:.3f} ms  {fl / ms_h / 1e9:.2f} TFLOP/s-equivalent  "
              f"{fl * (0.5 + 64 / n) / ms_h / 1e9:.2f} executed  maxrel {err:.1e}", flush=True)
        ms_t = t(lambda: torch.matmul(a, b, out=c))
        print(f"[cublas] zgemm {n}: {ms_t:.3f} ms  {fl / ms_t / 1e9:.2f} TFLOP/s", flush=True)
        # batched mid-size
        nb, bb = 1024, 16
        x = torch.randn(bb, nb, nb, dtype=torch.complex128, device="cuda")
        y = torch.randn(bb, nb, nb, dtype=torch.complex128, device="cuda")
        z = torch.empty_like(x)
        ms_b = t(lambda: lib.qch_zgemm_batched(_lib.dptr(x), _lib.dptr(y), _lib.dptr(z), nb, nb, nb, bb, nb * nb,
                                               nb * nb, nb * nb, sp))
        print(f"[{label}] zgemm {bb}x{nb}: {ms_b:.3f} ms  {bb * 8.0 * nb**3 / ms_b / 1e9:.2f} TFLOP/s", flush=True)
        ms_bt = t(lambda: torch.bmm(x, y, out=z))
        print(f"[cublas] zgemm {bb}x{nb}: {ms_bt:.3f} ms  {bb * 8.0 * nb**3 / ms_bt / 1e9:.2f} TFLOP/s", flush=True)


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    if os.environ.get("QCH_ZGEMM") == "cpasync":
        run(n, reps, "cpasync")
    else:
        run(n, reps, "tma")
        env = dict(os.environ, QCH_ZGEMM="cpasync")
        subprocess.run([sys.executable, __file__, str(n), str(reps)], env=env, check=False)
