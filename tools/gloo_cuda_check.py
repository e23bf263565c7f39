"""Which torch.distributed ops the gloo backend accepts for CUDA tensors
(used to dry-run bench.py's multi-rank paths with every rank on one GPU)."""
import os
import sys

import torch
import torch.distributed as dist


def main():
    rank = int(os.environ["RANK"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    x = torch.ones(4, dtype=torch.complex128, device="cuda") * (rank + 1)
    res = {}
    for name, fn in (
        ("all_reduce", lambda: dist.all_reduce(torch.ones(1, dtype=torch.float64, device="cuda"))),
        ("all_gather", lambda: dist.all_gather([torch.empty_like(x) for _ in range(2)], x)),
        ("all_gather_into_tensor", lambda: dist.all_gather_into_tensor(torch.empty(8, dtype=x.dtype, device="cuda"), x)),
        ("barrier", lambda: dist.barrier()),
        ("send_recv", lambda: dist.send(x, 1) if rank == 0 else dist.recv(x, 0)),
    ):
        try:
            fn()
            torch.cuda.synchronize()
            res[name] = "ok"
        except Exception as e:  # noqa: BLE001
            res[name] = f"FAIL {type(e).__name__}: {str(e)[:80]}"
    print(rank, res, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
