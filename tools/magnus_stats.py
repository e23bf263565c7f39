"""Phase counters of the fused Magnus kernel (QCH_MAGNUS_STATS): where the
cycles of one tile go.  python tools/magnus_stats.py [intervals ...]"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["QCH_MAGNUS_STATS"] = "1"


def main():
    import paper_2411_09982_b200 as eff
    from paper_2411_09982_b200 import _lib
    from paper_2411_09982_b200 import magnus as mg

    for m in [int(x) for x in sys.argv[1:]] or [100_000]:
        ch, grid = eff.driven_transmon(3, intervals=m, sub=4)
        d_psi = _lib.to_device(np.array([1, 0, 0], dtype=complex))
        for order in (2, 1):
            print(f"== M={m} order={order}", file=sys.stderr, flush=True)
            for _ in range(4):
                mg.evolve_device(ch, grid, m, d_psi, check=False, order=order)


if __name__ == "__main__":
    main()
