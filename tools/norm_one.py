"""qch_expm_norm_c128 (rownorm_kernel) over a batch of B N x N matrices:
time per launch (CUDA events) and GB/s.  argv: N B (one launch, for ncu) or
no argv: a sweep of N."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def run(n, b, reps=5):
    import torch

    from paper_2411_09982_b200 import _lib

    h = torch.randn((b, n, n), dtype=torch.complex128, device="cuda")
    out = torch.empty(b, dtype=torch.float64, device="cuda")
    f = lambda: _lib.load().qch_expm_norm_c128(_lib.dptr(h), b, n, _lib.dptr(out), _lib.stream_ptr())
    for _ in range(2):
        assert f() == 0
    torch.cuda.synchronize()
    if reps == 0:
        return
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"N={n:5d} B={b:5d}: {ms:8.3f} ms, {b * n * n * 16 / ms / 1e6:7.0f} GB/s, {ms * 1e3 / b:8.2f} us/matrix",
          flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 2048, reps=0)
    else:
        for n, b in ((64, 8192), (256, 2048), (1000, 128), (1024, 128), (2048, 32), (4096, 8)):
            run(n, b)
