"""Whole-GPU single-chain NPAD (npad_coop.cu): per-rotation time vs the
number of CTAs.  QCH_NPAD_COOP_CTAS=G python tools/coop_g_probe.py n_q n_r iters"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2411_09982_b200 as eff

    nq, nr, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    h = eff.transmon_resonator_hamiltonian(nq, nr).data
    op = eff.HermitianOperator(h)
    op.device_tensor()
    eff.npad_run(op, tol=1e-12, max_iter=min(iters, 1000))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = eff.npad_run(op, tol=1e-12, max_iter=iters)
    dt = time.perf_counter() - t0
    print(f"dim {nq * nr} applied {st.applied} converged {st.converged}: {dt / st.applied * 1e6:.2f} us/rot")


if __name__ == "__main__":
    main()
