"""Run ONE instance of a hot-path workload (after a warm-up) so ncu can
capture its kernels:  python tools/prof_driver.py <case> [arg]
cases: npad60 | npad4096 [max_iter] | sweep [points] | magnus2 [intervals] | magnus4096 | zgemm4096 | herm4096 | herm256
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import magnus as mg
    from paper_2411_09982_b200 import npad as npd

    case = sys.argv[1]
    arg = int(sys.argv[2]) if len(sys.argv) > 2 else None
    if case == "npad60":
        op = eff.HermitianOperator(eff.transmon_resonator_hamiltonian(3, 20).data)
        for _ in range(2):
            st = eff.npad_run(op, tol=1e-12)
        print("applied", st.applied)
    elif case == "npad4096":
        op = eff.HermitianOperator(eff.transmon_resonator_hamiltonian(4, 1024).data, validate=False)
        import time as _t
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = _t.perf_counter()
            st = eff.npad_run(op, tol=1e-12, max_iter=arg or 2000)
            torch.cuda.synchronize()
            dt = _t.perf_counter() - t0
        print("applied", st.applied, f"us/rot {dt / max(st.applied, 1) * 1e6:.2f}")
    elif case == "sweep":
        pts = eff.sweep_points(32, 32)[: (arg or 64)]
        for _ in range(2):
            res = npd.npad_sweep_transmon(pts, 4, 256, eff.sweep_target(256), tol=1e-12)
        print("rotations", int(res.applied.sum()))
    elif case == "sweepscale":
        # per-chain rotation latency vs number of concurrent chains
        from paper_2411_09982_b200 import _lib as lib
        allpts = eff.sweep_points(32, 32)
        for p in (1, 8, 74, 148, 296, 592, 1024):
            pts = allpts[:p]
            mats = npd.build_transmon_resonator_batch(pts, 4, 256)
            mx = torch.empty(p, dtype=torch.float64, device="cuda")
            for k in range(p):
                lib.call("qch_max_abs_c128", lib.dptr(mats[k]), 1024 * 1024, lib.dptr(mx[k:k + 1]), lib.stream_ptr())
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            ap, cv = npd._run_batch_inplace(mats, eff.sweep_target(256), 1e-12, None, mx)
            s1.record()
            torch.cuda.synchronize()
            ms = s0.elapsed_time(s1)
            rot = int(ap.sum().item())
            mx_rot = int(ap.max().item())
            print(f"points={p:5d} rotations={rot:7d} max_chain={mx_rot:4d} ms={ms:8.3f} "
                  f"rot/s={rot / ms * 1e3:.3e} us/rot(longest chain)={ms * 1e3 / mx_rot:.2f}")
    elif case == "magnus2":
        m = arg or 100000
        ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
        psi0 = torch.tensor([1, 0, 0], dtype=torch.complex128, device="cuda")
        for _ in range(2):
            tr = mg.evolve_device(ch, grid, m, psi0, check=False, order=2)
        torch.cuda.synchronize()
        print("traj", tr.shape)
    elif case == "givens":
        n = arg or 10**7
        op = eff.ladder_test_hamiltonian_device(n)
        st0 = eff.NPADState.from_operator(op)
        for _ in range(2):
            out = eff.eliminate_coupling(st0, 0, 1)
        print("nnz", out.current.nnz)
    elif case == "magnus4096":
        ch = eff.heisenberg_chain_hamiltonians(12)
        full = eff.synthetic_transfer_pulse(25.0, 4096 * 8 + 1, seed=7)
        grid = eff.ControlGrid(0.0, 25.0 / 4096, full.signals[:, :9])
        psi0 = np.zeros(4096, dtype=complex)
        psi0[0] = 1
        tr = mg.evolve_device(ch, grid, 1, torch.from_numpy(psi0).cuda(), check=False, order=2)
        torch.cuda.synchronize()
        print("traj", tr.shape)
    elif case in ("zgemm4096", "herm4096"):
        from paper_2411_09982_b200 import _lib as lib

        n = 4096
        a = torch.randn(n, n, dtype=torch.complex128, device="cuda")
        h = (a + a.mH) * 0.5
        c = torch.empty_like(a)
        for _ in range(2):
            if case == "zgemm4096":
                lib.call("qch_zgemm_batched", lib.dptr(h), lib.dptr(a), lib.dptr(c), n, n, n, 1, n * n, n * n, n * n,
                         lib.stream_ptr())
            else:
                lib.call("qch_zgemm_herm_batched", lib.dptr(h), lib.dptr(h), lib.dptr(c), n, 1, lib.stream_ptr())
        print(case, "done")
    elif case == "herm256":  # the mid-size line's Hermitian products: 2048 x (256 x 256) on DMMA
        from paper_2411_09982_b200 import _lib as lib

        n, b = 256, 2048
        a = torch.randn(b, n, n, dtype=torch.complex128, device="cuda")
        h = (a + a.mH) * 0.5
        c = torch.empty_like(a)
        for _ in range(2):
            lib.call("qch_zgemm_herm_batched", lib.dptr(h), lib.dptr(h), lib.dptr(c), n, b, lib.stream_ptr())
        print(case, "done")
    elif case == "oz4096":
        from paper_2411_09982_b200 import _lib as lib

        n = 4096
        a = torch.randn(n, n, dtype=torch.complex128, device="cuda")
        h = (a + a.mH) * 0.5
        c = torch.empty((8, n, n), dtype=torch.complex128, device="cuda")
        hb = h.expand(8, n, n).contiguous()
        for _ in range(2):
            lib.call("qch_zgemm_herm_batched", lib.dptr(hb), lib.dptr(hb), lib.dptr(c), n, 8, lib.stream_ptr())
        print(case, "done")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
