"""Convergence curves on the device (BASELINE.json configs[0], [1], [2]).

* Kuhn poker: EGT/as and CFR+ until eps_sad <= 1e-6 (iterations, device seconds).
* Leduc hold'em: EGT (Alg. 1), EGT with mu balancing, EGT/as (Alg. 3-4) against CFR(RM),
  CFR(RM+) and CFR+ -- eps_sad after 1, 3, 10, ..., 10000 iterations (PAPER.md:705-716 plots
  the same quantity against gradient evaluations; EGT does 3 or 4 per iteration, CFR 2).
* One synthetic NLHE river subgame with the {1/2, 1, all-in} abstraction: EGT/as against CFR+,
  eps_sad in mbb of the 100-chip big blind.

Everything runs through the public API (binding -> C ABI -> CUDA); EGT's mu comes from the
library's practical search (R14).  Device time is CUDA-event time of the iterations
(the gap evaluations between checkpoints are excluded).  Writes JSON lines and, with --md, a
markdown summary.

    python tools/convergence.py --md profiles/r01_convergence.md
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHECKPOINTS = [1, 3, 10, 30, 100, 300, 1000, 3000, 10000]
GRADS_PER_ITER = {"egt": 3, "egt_balanced": 3, "egt_as": 4, "cfr_rm": 2, "cfr_rmp": 2, "cfr_plus": 2}


def curve(P, game, solver, checkpoints, stream):
    import torch
    from paper_1810_03063_b200.solve import SOLVERS
    kind, code = SOLVERS[solver]
    if kind == "egt":
        game.egt_init(code)
        step, which = game.egt_step, 0
    else:
        game.cfr_init(code)
        step, which = game.cfr_step, 1
    pts, done, secs = [], 0, 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for c in checkpoints:
        e0.record(stream)
        step(c - done)
        e1.record(stream)
        e1.synchronize()
        secs += e0.elapsed_time(e1) / 1e3
        done = c
        gap = float(game.saddle_gap(which).max())
        pts.append({"iters": c, "grad_evals": c * GRADS_PER_ITER[solver], "gap": gap, "device_s": secs})
    return pts


def to_eps(P, game, solver, eps, max_iters, stream, every=10):
    import torch
    from paper_1810_03063_b200.solve import SOLVERS
    kind, code = SOLVERS[solver]
    if kind == "egt":
        game.egt_init(code)
        step, which = game.egt_step, 0
    else:
        game.cfr_init(code)
        step, which = game.cfr_step, 1
    it, secs = 0, 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gap = float("inf")
    while it < max_iters and gap > eps:
        n = max(every, it // 50)  # checks every ~2 % of the run (at least every `every` iterations)
        e0.record(stream)
        step(n)
        e1.record(stream)
        e1.synchronize()
        secs += e0.elapsed_time(e1) / 1e3
        it += n
        gap = float(game.saddle_gap(which).max())
    return {"solver": solver, "eps": eps, "iters": it, "gap": gap, "device_s": secs, "reached": gap <= eps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-leduc", type=int, default=10000)
    ap.add_argument("--river-iters", type=int, default=3000)
    ap.add_argument("--seed", type=int, default=2100)
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    import torch
    import paper_1810_03063_b200 as P
    from paper_1810_03063_b200 import workloads as W
    stream = torch.cuda.Stream()
    out = {"kuhn": [], "leduc": {}, "river": {}}

    for solver in ("egt_as", "cfr_plus"):
        g = P.Game(P.KUHN, n_games=1)
        g.set_stream(stream)
        r = to_eps(P, g, solver, 1e-6, 2000000, stream)
        out["kuhn"].append(r)
        print(json.dumps({"game": "kuhn", **r}), flush=True)
        g.close()

    cps = [c for c in CHECKPOINTS if c <= a.max_leduc]
    for solver in ("egt", "egt_balanced", "egt_as", "cfr_rm", "cfr_rmp", "cfr_plus"):
        g = P.Game(P.LEDUC, n_games=1)
        g.set_stream(stream)
        pts = curve(P, g, solver, cps, stream)
        out["leduc"][solver] = pts
        print(json.dumps({"game": "leduc", "solver": solver, "curve": pts}), flush=True)
        g.close()

    spec = W.river_spec("simple")
    boards = W.random_boards(1, a.seed)
    p1, p2 = W.random_priors(boards, a.seed)
    rcps = [c for c in CHECKPOINTS if c <= a.river_iters] + ([a.river_iters] if a.river_iters not in CHECKPOINTS else [])
    for solver in ("egt_as", "cfr_plus"):
        g = P.Game(P.RIVER, n_games=1, river=spec, boards=boards, prior1=p1, prior2=p2)
        g.set_stream(stream)
        pts = curve(P, g, solver, rcps, stream)
        for q in pts:
            q["gap_mbb"] = q["gap"] / 100.0 * 1000.0
        out["river"][solver] = pts
        print(json.dumps({"game": "river_simple", "solver": solver, "curve": pts}), flush=True)
        g.close()

    if a.md:
        L = ["# Convergence on one B200 (BASELINE.json configs[0]-[2])", "",
             "`python tools/convergence.py` -- public API, CUDA graphs; eps_sad = max_y x^T A y - min_x x^T A y "
             "(PAPER.md:311) of the EGT iterate / the CFR average; device seconds exclude the gap checks.", "",
             "## Kuhn poker to eps_sad <= 1e-6 (configs[0]; game value -1/18 is checked in tests/test_gpu_api.py)", "",
             "| solver | iterations | eps_sad | device s |", "|---|---|---|---|"]
        for r in out["kuhn"]:
            L.append("| %s | %d | %.2e | %.4f |" % (r["solver"], r["iters"], r["gap"], r["device_s"]))
        L += ["", "## Leduc hold'em: eps_sad after t iterations (configs[1])", "",
              "| iterations | " + " | ".join(out["leduc"]) + " |", "|---|" + "---|" * len(out["leduc"])]
        for i, c in enumerate(cps):
            L.append("| %d | " % c + " | ".join("%.3e" % out["leduc"][s][i]["gap"] for s in out["leduc"]) + " |")
        L += ["", "Gradient evaluations per iteration: EGT 3, EGT/as 4 (incl. the excessive-gap check), CFR 2; "
              "device seconds at the last checkpoint: " +
              ", ".join("%s %.3f" % (s, out["leduc"][s][-1]["device_s"]) for s in out["leduc"]) + ".", "",
              "## River subgame, {1/2, 1, all-in} abstraction, 1081 x 1081 hands (configs[2]): eps_sad in mbb", "",
              "| iterations | " + " | ".join(out["river"]) + " |", "|---|" + "---|" * len(out["river"])]
        for i, c in enumerate(rcps):
            L.append("| %d | " % c + " | ".join("%.2f" % out["river"][s][i]["gap_mbb"] for s in out["river"]) + " |")
        L += ["", "Device seconds at the last checkpoint: " +
              ", ".join("%s %.3f" % (s, out["river"][s][-1]["device_s"]) for s in out["river"]) + "."]
        with open(a.md, "w") as f:
            f.write("\n".join(L) + "\n")


if __name__ == "__main__":
    main()
