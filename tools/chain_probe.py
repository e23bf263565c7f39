"""Ordered-product (qch_magnus_chain_c128) time per interval vs N, for the
kernel QCH_CHAIN_CLUSTER_MAX selects.  python tools/chain_probe.py"""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2411_09982_b200 import _lib

    lib = _lib.load()
    tag = os.environ.get("QCH_CHAIN_CLUSTER_MAX", "default")
    for n in [int(v) for v in os.environ.get("CHAIN_NS", "96,128,192,256,320,384,512,768").split(",")]:
        m = 2048 if n <= 512 else 512 if n <= 1024 else 64
        u = torch.randn((m, n, n), dtype=torch.complex128, device="cuda")
        u = torch.linalg.qr(u)[0]
        psi = torch.zeros(n, dtype=torch.complex128, device="cuda")
        psi[0] = 1
        rows = torch.empty((m, n), dtype=torch.complex128, device="cuda")
        bad = ctypes.c_int64(-1)
        args = (_lib.dptr(u), n, m, _lib.dptr(psi), _lib.dptr(rows), ctypes.byref(bad), _lib.stream_ptr())
        for _ in range(3):
            assert lib.qch_magnus_chain_c128(*args) == 0, _lib.last_error()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            lib.qch_magnus_chain_c128(*args)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"[{tag}] N={n:4d} M={m}: {ms:8.3f} ms, {ms * 1e3 / m:6.3f} us/interval", flush=True)
        del u, rows


if __name__ == "__main__":
    main()
