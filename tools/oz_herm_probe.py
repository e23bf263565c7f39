"""Hermitian int8 (Ozaki) product probe at the config-5 shape: n = 4096,
batch 8, C = A A through qch_zgemm_herm_batched, per-kernel times.
python tools/oz_herm_probe.py [reps]   (ncu: -k regex:oz_gemm --launch-skip 3 -c 1)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2411_09982_b200 import _lib

    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    n, b = 4096, 8
    a = torch.randn(b, n, n, dtype=torch.complex128, device="cuda")
    a = (a + a.transpose(1, 2).conj()) / 2
    c = torch.empty_like(a)
    call = lambda: _lib.call("qch_zgemm_herm_batched", _lib.dptr(a), _lib.dptr(a), _lib.dptr(c), n, b,  # noqa: E731
                             _lib.stream_ptr())
    call()
    torch.cuda.synchronize()
    _lib.profile_read(reset=True)
    _lib.profile_enable(True)
    o0 = _lib.load().qch_int8_ops()
    for _ in range(reps):
        call()
    torch.cuda.synchronize()
    _lib.profile_enable(False)
    ops = _lib.load().qch_int8_ops() - o0
    prof = _lib.profile_read(reset=True)
    for k, (ms, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:24s} {ms / reps:9.3f} ms/product  x{cnt}")
    g = prof["oz_gemm"][0] * 1e-3
    print(f"int8 TOPS in oz_gemm: {ops / g / 1e12:.1f}")


if __name__ == "__main__":
    main()
