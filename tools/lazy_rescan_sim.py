"""How often would lazy row rescans be needed? (config-3 analysis, host)
Follows the exact greedy chain (oracle run_incremental's row maxima) and, on
the side, a lazy variant: a row whose best was rotated keeps an upper bound
instead of being rescanned; a selection needs a resolution (rescans + one
more exchange) only when some lazy bound could reach the pivot.
python tools/lazy_rescan_sim.py [n_q n_r steps]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    from oracle import npad_oracle as no
    import paper_2411_09982_b200.models as models

    nq, nr, steps = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (4, 1024, 3000)
    h = np.array(models.transmon_resonator_hamiltonian(nq, nr).data, dtype=np.complex128)
    n = h.shape[0]
    rm = no._RowMax(h, None)
    lazy = np.zeros(n, dtype=bool)
    bound = np.zeros(n)
    rescans_eager = 0
    resolutions = 0
    rescans_lazy = 0
    for step in range(steps):
        pick = rm.best()
        if pick is None:
            break
        i, j, mag = pick
        # lazy selection: exact rows only (lazy rows' true values are in rm, but the lazy scheme does not know them)
        ex = ~lazy
        ex[[i, j]] = True
        vals = np.where(ex, rm.val, -1.0)
        pbest = vals.max()
        if (lazy & (bound >= pbest * (1 - 1e-12))).any():
            resolutions += 1
            hit = lazy & (bound >= pbest * (1 - 1e-12))
            rescans_lazy += int(hit.sum())
            lazy[hit] = False
        # rotate
        c, sh, ph, _ = no.rotation_scalars(h, i, j)
        no.rotate(h, i, j, c, no.block_s(sh, ph))
        # eager: rows with best column in {i, j}
        stale = np.flatnonzero(((rm.col == i) | (rm.col == j)) & (np.arange(n) != i) & (np.arange(n) != j))
        rescans_eager += stale.size
        old = rm.val.copy()
        rm.after_rotation(i, j)
        # lazy bookkeeping: stale rows become lazy with bound = old best (others unchanged) max the new entries
        for x in stale:
            if not lazy[x]:
                lazy[x] = True
                bound[x] = old[x]
        # lazy rows: entries at columns i, j changed -> bound grows to cover them
        for cidx in (i, j):
            xs = np.flatnonzero(lazy)
            xs = xs[xs > cidx]
            if xs.size:
                bound[xs] = np.maximum(bound[xs], np.abs(h[xs, cidx]))
        lazy[[i, j]] = False  # pivot rows: exact from the partials
    print(f"dim {n}, {step + 1} rotations: eager rescans {rescans_eager / (step + 1):.3f}/rotation; lazy: "
          f"resolution rounds {resolutions / (step + 1):.3f}/rotation, rescans {rescans_lazy / (step + 1):.3f}/rotation, "
          f"lazy rows at the end {int(lazy.sum())}")


if __name__ == "__main__":
    main()
