"""One qch_expm_norm_c128 launch over a batch of B N x N matrices (argv: N B)
for ncu captures of rownorm_kernel."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2411_09982_b200 import _lib

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    h = torch.randn((b, n, n), dtype=torch.complex128, device="cuda")
    out = torch.empty(b, dtype=torch.float64, device="cuda")
    for _ in range(2):
        assert _lib.load().qch_expm_norm_c128(_lib.dptr(h), b, n, _lib.dptr(out), _lib.stream_ptr()) == 0
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
