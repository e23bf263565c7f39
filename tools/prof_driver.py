"""Run ONE instance of a hot-path workload (after a warm-up) so ncu can
capture its kernels:  python tools/prof_driver.py <case> [arg]
cases: npad60 | npad4096 [max_iter] | sweep [points] | magnus2 [intervals] | magnus4096
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
        for _ in range(2):
            st = eff.npad_run(op, tol=1e-12, max_iter=arg or 2000)
        print("applied", st.applied)
    elif case == "sweep":
        pts = eff.sweep_points(8, (arg or 64) // 8)
        for _ in range(2):
            res = npd.npad_sweep_transmon(pts, 4, 256, eff.sweep_target(256), tol=1e-12)
        print("rotations", int(res.applied.sum()))
    elif case == "magnus2":
        m = arg or 100000
        ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
        psi0 = torch.tensor([1, 0, 0], dtype=torch.complex128, device="cuda")
        for _ in range(2):
            tr = mg.evolve_device(ch, grid, m, psi0, check=False, order=2)
        torch.cuda.synchronize()
        print("traj", tr.shape)
    elif case == "magnus4096":
        ch = eff.heisenberg_chain_hamiltonians(12)
        full = eff.synthetic_transfer_pulse(25.0, 4096 * 8 + 1, seed=7)
        grid = eff.ControlGrid(0.0, 25.0 / 4096, full.signals[:, :9])
        psi0 = np.zeros(4096, dtype=complex)
        psi0[0] = 1
        tr = mg.evolve_device(ch, grid, 1, torch.from_numpy(psi0).cuda(), check=False, order=2)
        torch.cuda.synchronize()
        print("traj", tr.shape)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
