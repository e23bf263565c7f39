"""tcgen05 int8 GEMM probe: correctness vs an exact integer reference and
throughput.  python tools/i8gemm_probe.py"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2411_09982_b200 import _lib

    lib = _lib.load()
    fn = lib.qch_i8gemm_test
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 3 + [ctypes.c_void_p]
    g = torch.Generator().manual_seed(0)
    for m, n, k in [(128, 128, 128), (128, 128, 256), (256, 384, 512), (200, 136, 160), (1024, 1024, 4096)]:
        a = torch.randint(-127, 128, (m, k), generator=g, dtype=torch.int8)
        b = torch.randint(-127, 128, (n, k), generator=g, dtype=torch.int8)
        ref = (a.double() @ b.double().T).round().long()
        da, db = a.cuda(), b.cuda()
        dc = torch.zeros(m, n, dtype=torch.int32, device="cuda")
        rc = fn(da.data_ptr(), db.data_ptr(), dc.data_ptr(), m, n, k, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        got = dc.cpu().long()
        bad = (got != ref).sum().item()
        print(f"{m}x{n}x{k}: rc={rc} mismatches={bad}", flush=True)
        if bad:
            idx = (got != ref).nonzero()[:4]
            print("   first bad", [(int(i), int(j), int(got[i, j]), int(ref[i, j])) for i, j in idx.tolist()])
    n = 4096
    a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    c = torch.empty(n, n, dtype=torch.int32, device="cuda")
    for kk in (4096, 8 * 4096):
        if kk > n:
            a2 = torch.randint(-127, 128, (n, kk), dtype=torch.int8, device="cuda")
            b2 = torch.randint(-127, 128, (n, kk), dtype=torch.int8, device="cuda")
        else:
            a2, b2 = a, b
        fn(a2.data_ptr(), b2.data_ptr(), c.data_ptr(), n, n, kk, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            fn(a2.data_ptr(), b2.data_ptr(), c.data_ptr(), n, n, kk, torch.cuda.current_stream().cuda_stream)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        print(f"4096x4096x{kk}: {ms:.3f} ms  {2.0 * n * n * kk / ms / 1e9:.1f} TOPS", flush=True)


if __name__ == "__main__":
    main()
