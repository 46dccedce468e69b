"""User-facing driver: solve a batch of endgames to a target saddle-point gap.

Argument marshalling and the stopping loop only -- every iteration, gradient, treeplex
pass and gap evaluation runs in the CUDA library through the C ABI (include/egt_b200.h).
The loop is Alg. 3's "while eps_sad(x^t, y^t) > eps" evaluated every
``check_every`` iterations on the device (one small device-to-host copy per check).
"""
import numpy as np

from . import binding as B

SOLVERS = {"egt": ("egt", B.EGT_THEORY), "egt_balanced": ("egt", B.EGT_BALANCED), "egt_as": ("egt", B.EGT_AS),
           "cfr_rm": ("cfr", B.CFR_RM), "cfr_rmp": ("cfr", B.CFR_RMP), "cfr_plus": ("cfr", B.CFR_PLUS)}


def solve(game, solver="egt_as", eps=None, eps_mbb=None, max_iters=10000, check_every=10, mu=None):
    """Run `solver` on every game of `game` (a binding.Game) until each game's eps_sad <= eps
    (in the game's payoff unit; river games: chips, or give eps_mbb with the big blind of 100
    chips) or max_iters.  mu: initial smoothing for EGT (None: the practical
    search, R14).  Returns {"gap": per-game eps_sad (host fp64), "iters": iterations
    run, "strategy": (x, y) -- the EGT iterate or the CFR average, sequence form, host fp64
    [n_games, n_pub, n_combos] in canonical hand order}."""
    if solver not in SOLVERS:
        raise ValueError("solver must be one of %s" % sorted(SOLVERS))
    if eps_mbb is not None:
        eps = eps_mbb * 100.0 / 1000.0
    if eps is None:
        eps = 0.0
    kind, code = SOLVERS[solver]
    if kind == "egt":
        if mu is None:
            game.egt_init(code)
        else:
            game.egt_init(code, mu, mu)
        step, which = game.egt_step, 0
    else:
        game.cfr_init(code)
        step, which = game.cfr_step, 1
    use_target = eps > 0 and (kind == "cfr" or solver == "egt_as")
    if use_target:
        game.egt_set_target(eps)  # solved games stop on the device (no work spent on them)
    # at least one iteration first: the CFR average is defined from iteration 1 on
    # (Gen-CFR line 34 with alpha^1 = 1)
    it = min(check_every, max_iters) if max_iters > 0 else 0
    if it:
        step(it)
    gap = game.saddle_gap(which)
    while it < max_iters and np.max(gap) > eps:
        n = min(check_every, max_iters - it)
        step(n)
        it += n
        gap = game.saddle_gap(which)
    if use_target:
        game.egt_set_target(None)
    strategy = (game.get_avg_strategy(0), game.get_avg_strategy(1))
    return {"gap": gap, "iters": it, "strategy": strategy}
