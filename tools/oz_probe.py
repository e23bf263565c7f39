"""Ozaki (int8 tcgen05) real GEMM probe: accuracy vs FP64 and throughput.
python tools/oz_probe.py"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2411_09982_b200 import _lib

    lib = _lib.load()
    fn = lib.qch_oz_real_test
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                   ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
    sp = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    rng = np.random.default_rng(0)
    for m, n, k in [(128, 128, 128), (256, 384, 512), (200, 136, 160), (1024, 1024, 4096)]:
        x = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
        y = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
        x[3] *= 1e-5  # rows of very different scale
        dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        for xc, yc, ref in ((0, 0, x.real @ y.real.T), (1, 4, x.imag @ (-y.imag).T), (2, 3, (x.real + x.imag) @ (y.real - y.imag).T)):
            for s in (6, 7, 8):
                out = torch.zeros(m, n, dtype=torch.float64, device="cuda")
                rc = fn(dx.data_ptr(), xc, dy.data_ptr(), yc, out.data_ptr(), m, n, k, s, sp())
                torch.cuda.synchronize()
                got = out.cpu().numpy()
                scale = np.abs(x).max(axis=1)[:, None] * np.abs(y).max(axis=1)[None, :] * k
                err = np.abs(got - ref) / scale
                rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
                print(f"{m}x{n}x{k} comp {xc},{yc} s={s}: rc={rc} max err/scale {err.max():.2e} rel fro {rel:.2e}",
                      flush=True)
    n = 4096
    x = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    out = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for s in (7,):
        fn(x.data_ptr(), 0, x.data_ptr(), 0, out.data_ptr(), n, n, n, s, sp())
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(3):
            fn(x.data_ptr(), 0, x.data_ptr(), 0, out.data_ptr(), n, n, n, s, sp())
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 3
        print(f"real 4096^3 s={s}: {ms:.3f} ms incl. slicing -> {2 * n**3 / ms / 1e9:.1f} FP64-equivalent TFLOP/s; "
              f"int8 {s * (s + 1) / 2 * 2 * n**3 / ms / 1e9:.0f} TOPS", flush=True)


if __name__ == "__main__":
    main()
