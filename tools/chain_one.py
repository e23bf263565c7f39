"""One ordered-product launch at N (argv[1], default 128) for ncu captures."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2411_09982_b200 import _lib

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    lib = _lib.load()
    u = torch.linalg.qr(torch.randn((m, n, n), dtype=torch.complex128, device="cuda"))[0]
    psi = torch.zeros(n, dtype=torch.complex128, device="cuda")
    psi[0] = 1
    rows = torch.empty((m, n), dtype=torch.complex128, device="cuda")
    bad = ctypes.c_int64(-1)
    for _ in range(2):
        assert lib.qch_magnus_chain_c128(_lib.dptr(u), n, m, _lib.dptr(psi), _lib.dptr(rows), ctypes.byref(bad),
                                         _lib.stream_ptr()) == 0, _lib.last_error()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
