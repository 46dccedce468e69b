"""One EGT/as iteration on a bench-shaped batch, for ncu captures (not a benchmark).

Loads --batch Libratus-scale endgames, initialises EGT/as with an explicit mu (no search:
6 treeplex + 5 gradient launches), then runs --steps eager iterations (timing mode, so every
kernel is a separate launch).  Kernel order per iteration: prepare, [combine, grad, SBR+comb,
grad, prox] x 2 players (masked), 2 x (grad, SBR), 2 x BR, accept."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=148)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--precision", default="f64")
    ap.add_argument("--mu", type=float, default=20.0)
    a = ap.parse_args()
    import torch
    import paper_1810_03063_b200 as P
    args = type("A", (), {"workload": "libratus", "seed": 2100, "batch": a.batch})()
    spec, boards, p1, p2 = bench.workload(args, 0)
    G = P.Game(P.RIVER, n_games=a.batch, river=spec, boards=boards, prior1=p1, prior2=p2, precision=a.precision)
    G.egt_init(P.EGT_AS, a.mu, a.mu)
    G.timing(True)
    G.egt_step(a.steps)
    kt = G.timing_get()
    torch.cuda.synchronize()
    print({k: round(v[0], 3) for k, v in kt.items()})


if __name__ == "__main__":
    main()
