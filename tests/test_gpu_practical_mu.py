"""Parity at the bench's operating point: EGT/as from the practical mu (reading R14).

egt_init(EGT_AS) with mu <= 0 scans k = 0, 1, ... (mu = mu_theory * 2^-k) on the device; the
oracle's egt.practical_mu scans the same k on the CPU, so the chosen k must be the same integer
per game, and from there every EGT/as attempt (Alg. 3-4) -- accept or
backtrack, mu, tau, iterate, eps_sad -- must match attempt by attempt.  At this mu the smoothed
responses' behavioural probabilities underflow within a few iterations: the prox centres are
carried as behavioural logs on both sides (reading R16).

The oracle is stepped one ATTEMPT at a time (a failed excessive-gap check halves tau and keeps
the iterate, Alg. 4), composed from its own primitives egt.step_xy and egt.excessive_gap.
"""
import concurrent.futures as cf
import multiprocessing as mp

import numpy as np
import pytest

from oracle import br, egt
from tests.paritylib import Pair, assert_parity, assert_scalar

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-9


class _Perturbed(egt.Problem):
    """The same problem with every gradient perturbed by 1e-16 * max|g| per entry (about half
    an ulp of the largest entry: what a different, equally valid summation order changes).
    The spread between a perturbed and an unperturbed oracle run is the problem's own
    sensitivity to rounding; at a small smoothing mu the smoothed responses amplify gradient
    rounding by ~|g| / (mu beta), so deep into EGT/as the two runs drift apart by more than
    1e-9 although both are correct to rounding."""

    def __init__(self, sf, seed):
        super().__init__(sf)
        self.rng = np.random.default_rng(seed)

    def grad(self, v, other):
        g = super().grad(v, other)
        return g + 1e-16 * np.abs(g).max() * self.rng.standard_normal(g.shape)


class Attempts:
    """EGT/as (Alg. 3 with Alg. 4 unrolled: one Step + EGC check per attempt) on the oracle."""

    def __init__(self, sf, mu, perturb=None):
        self.sf = sf
        self.prob = egt.Problem(sf) if perturb is None else _Perturbed(sf, perturb)
        x, y = egt.initialize(self.prob, mu, mu)
        self.st = egt.EGTState(x, y, mu, mu)
        self.accepted = 0

    def attempt(self):
        st = self.st
        focus = "x" if st.mu_x > st.mu_y else "y"                  # Alg. 3 line 6
        mu_x, mu_y, x, y = egt.step_xy(self.prob, st, focus, st.tau)  # Alg. 4 line 1 / 4
        if egt.excessive_gap(self.prob, x, y, mu_x, mu_y) >= 0:    # Alg. 4 line 2 (R8)
            st.mu_x, st.mu_y, st.x, st.y = mu_x, mu_y, x, y
            self.accepted += 1
        else:
            st.tau *= 0.5                                          # Alg. 4 line 3
            st.backtracks += 1


def _strategies(G, which=0):
    out = []
    for p in (0, 1):
        d = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        G.get_strategy_device(p, which, d)
        torch.cuda.synchronize()
        out.append(d.cpu().numpy().reshape(G.n_games, -1))
    return out


def _compare(pair, g, sc, xs, ys, gap, run, what, pert=None):
    """Decisions (accepted steps, backtracks) exactly; mu, tau, iterate and eps_sad at 1e-9
    relative per element -- plus, when `pert` (a perturbed oracle run) is given, 30x the
    oracle's own sensitivity to rounding, max |oracle - perturbed oracle| (the trajectory's
    sensitivity is global: a rounding difference anywhere moves every entry)."""
    st = run.st
    assert int(sc[g, 3]) == run.accepted and int(sc[g, 5]) == st.backtracks, what
    if pert is not None:  # the spread is only meaningful along the same accept decisions
        assert pert.accepted == run.accepted and pert.st.backtracks == st.backtracks, what
    assert_scalar(sc[g, 0], st.mu_x, TOL, what + " mu", floor=0)
    assert_scalar(sc[g, 1], st.mu_y, TOL, what + " mu", floor=0)
    assert_scalar(sc[g, 2], st.tau, TOL, what + " tau", floor=0)
    for p, got, want in ((0, xs[g], st.x), (1, ys[g], st.y)):
        got = pair.from_product(g, p, got)[1:]
        if pert is None:
            assert_parity(got, want[1:], TOL, what + (" x", " y")[p])
        else:
            other = (pert.st.x, pert.st.y)[p][1:]
            spread = np.abs(other - want[1:])
            err = np.abs(got - want[1:])
            bound = TOL * np.abs(want[1:]) + 1e-13 * np.abs(want[1:]).max() + 30.0 * spread.max()
            assert np.all(err <= bound), (what, float(err.max()), float(spread.max()))
            REPORT_SENS[what] = max(REPORT_SENS.get(what, 0.0), float(spread.max()))
    want_gap = br.saddle_gap(pair.sf[g], st.x, st.y)
    floor = 1e-12 if pert is None else 1e-12 + 30.0 * abs(br.saddle_gap(pair.sf[g], pert.st.x, pert.st.y) - want_gap)
    assert_scalar(gap[g], want_gap, TOL, what + " eps_sad", floor=floor)


REPORT_SENS = {}


# ------------------------------------------------------------------ small games, many attempts
@pytest.mark.parametrize("case", [dict(kind="kuhn", n_games=1), dict(kind="leduc", n_games=1),
                                  dict(kind="river", n_games=3, seed=1),
                                  dict(kind="river", n_games=2, seed=8, n_ranks=6, n_suits=4)])
def test_practical_mu_egt_as_small(case):
    import paper_1810_03063_b200 as P
    pair = Pair(**case)
    G = pair.game
    G.egt_init(P.EGT_AS)
    sc = G.egt_scalars()
    runs, perts = {}, {}
    for g in range(G.n_games):
        k, mu = egt.practical_mu(pair.sf[g])
        assert_scalar(sc[g, 0], mu, 1e-14, "practical mu", floor=0)     # same k (mu is mu_th * 2^-k)
        assert_scalar(sc[g, 1], mu, 1e-14, "practical mu", floor=0)
        runs[g] = Attempts(pair.sf[g], mu)
        perts[g] = Attempts(pair.sf[g], mu, perturb=g + 1)
    n_bt = 0
    done = 0
    for n in (10, 25, 60):
        G.egt_step(n - done)
        for g in range(G.n_games):
            for _ in range(n - done):
                runs[g].attempt()
                perts[g].attempt()
        done = n
        sc = G.egt_scalars()
        xs, ys = _strategies(G)
        gap = G.saddle_gap(0)
        for g in range(G.n_games):
            assert int(sc[g, 4]) == n
            # first 10 attempts: the north star's 1e-9 per element; deeper, where mu has shrunk
            # and the oracle's own rounding spread exceeds it, within 30x that spread
            _compare(pair, g, sc, xs, ys, gap, runs[g], "practical egt/as[%s]" % pair.kind,
                     pert=None if n == 10 else perts[g])
    n_bt = sum(r.st.backtracks for r in runs.values())
    assert n_bt >= 1, "no backtrack exercised"


# ------------------------------------------------------------------ the bench batch
BENCH_BATCH = 296
N_ATTEMPTS = 30


def _oracle_job(job):
    """Runs in a worker process (the oracle is single-threaded numpy): ("scan", g) -> k;
    ("attempts", g, mu) -> the oracle state after N_ATTEMPTS attempts."""
    import bench
    from oracle import river
    from oracle.cards import Deck
    from paper_1810_03063_b200 import workloads as W
    args = type("A", (), {"workload": "libratus", "seed": 2100, "batch": BENCH_BATCH})()
    spec, boards, p1, p2 = bench.workload(args, 0)
    g = job[1]
    rp = river.RiverParams(**{k: spec[k] for k in ("pot", "stack", "fracs", "allin", "raise_cap", "open_fold")})
    sf = river.RiverSeqForm(rp, Deck(13, 4), boards[g], W.prior_dict(p1[g], 52), W.prior_dict(p2[g], 52),
                            build_sparse=False)
    if job[0] == "scan":
        return egt.practical_mu(sf)
    run = Attempts(sf, job[2], perturb=None if job[0] == "attempts" else 7)
    for _ in range(N_ATTEMPTS):
        run.attempt()
    st = run.st
    return dict(accepted=run.accepted, backtracks=st.backtracks, mu_x=st.mu_x, mu_y=st.mu_y, tau=st.tau,
                x=st.x, y=st.y, gap=br.saddle_gap(sf, st.x, st.y))


def test_practical_mu_bench_batch():
    """The 296-game bench batch in bench.py's launch configuration: the device scan picks the
    oracle's k on sampled games, then 30 graph-launched EGT/as attempts of the whole batch; a
    game with at least one backtrack among them is checked attempt-exactly against the oracle
    (oracle runs in worker processes, in parallel)."""
    import bench
    import paper_1810_03063_b200 as P
    args = type("A", (), {"workload": "libratus", "seed": 2100, "batch": BENCH_BATCH})()
    spec, boards, p1, p2 = bench.workload(args, 0)
    pair = Pair("river", n_games=BENCH_BATCH, spec=spec, boards=boards, priors=(p1, p2), sample=[],
                build_sparse=False)
    G = pair.game
    G.egt_init(P.EGT_AS)
    sc0 = G.egt_scalars()
    G.egt_step(N_ATTEMPTS)
    sc = G.egt_scalars()
    assert np.all(sc[:, 4] == N_ATTEMPTS)
    bt = np.flatnonzero(sc[:, 5] >= 1)
    g_bt = int(bt[0]) if len(bt) else 0
    sample = sorted({0, g_bt, BENCH_BATCH - 1})
    ctx = mp.get_context("spawn")
    with cf.ProcessPoolExecutor(max_workers=len(sample) + 1, mp_context=ctx) as ex:
        scans = {g: ex.submit(_oracle_job, ("scan", g)) for g in sample}
        att = ex.submit(_oracle_job, ("attempts", g_bt, float(sc0[g_bt, 0])))
        att_p = ex.submit(_oracle_job, ("perturbed", g_bt, float(sc0[g_bt, 0])))
        for g in sample:
            k, mu = scans[g].result()
            assert_scalar(sc0[g, 0], mu, 1e-14, "bench-batch practical mu", floor=0)
            assert_scalar(sc0[g, 1], mu, 1e-14, "bench-batch practical mu", floor=0)
        want = att.result()
        pert = att_p.result()
    xs, ys = _strategies(G)
    gap = G.saddle_gap(0)
    from oracle import river
    from oracle.cards import Deck
    from paper_1810_03063_b200 import workloads as W
    rp = river.RiverParams(**{k: spec[k] for k in ("pot", "stack", "fracs", "allin", "raise_cap", "open_fold")})
    sf = river.RiverSeqForm(rp, Deck(13, 4), boards[g_bt], W.prior_dict(p1[g_bt], 52),
                            W.prior_dict(p2[g_bt], 52), build_sparse=False)
    pair.sf[g_bt] = sf
    assert int(sc[g_bt, 3]) == want["accepted"] and int(sc[g_bt, 5]) == want["backtracks"]
    assert len(bt) == 0 or want["backtracks"] >= 1
    assert_scalar(sc[g_bt, 0], want["mu_x"], TOL, "bench-batch practical egt/as mu", floor=0)
    assert_scalar(sc[g_bt, 1], want["mu_y"], TOL, "bench-batch practical egt/as mu", floor=0)
    assert_scalar(sc[g_bt, 2], want["tau"], TOL, "bench-batch practical egt/as tau", floor=0)
    # 1e-9 per element, plus 30x the oracle's own rounding sensitivity (a perturbed oracle run,
    # see _Perturbed), which after 30 attempts at the practical mu is of the same order
    assert pert["accepted"] == want["accepted"] and pert["backtracks"] == want["backtracks"]
    for p, key in ((0, "x"), (1, "y")):
        got = pair.from_product(g_bt, p, (xs, ys)[p][g_bt])[1:]
        spread = float(np.abs(pert[key][1:] - want[key][1:]).max())
        err = np.abs(got - want[key][1:])
        bound = TOL * np.abs(want[key][1:]) + 1e-13 * np.abs(want[key][1:]).max() + 30.0 * spread
        assert np.all(err <= bound), (key, float(err.max()), spread)
        REPORT_SENS["bench-batch " + key] = spread
        assert_parity(got, want[key][1:], 1.0, "bench-batch practical egt/as " + key)  # records the worst rel. error
    assert_scalar(gap[g_bt], want["gap"], TOL, "bench-batch practical egt/as eps_sad",
                  floor=1e-12 + 30.0 * abs(pert["gap"] - want["gap"]))
    print("bench batch: game %d, %d backtracks in %d attempts; games with a backtrack: %d"
          % (g_bt, want["backtracks"], N_ATTEMPTS, len(bt)))


def test_egt_init_independent_of_previous_state():
    """egt_init with the practical mu on a game that already ran CFR, and a second egt_init on
    the same game, leave exactly the state a fresh game's egt_init does (no stale scratch: the
    mu scan's omega gradient writes every row; round 1 read an unwritten buffer there), and that
    state is the oracle's practical mu and initial point (Alg. 3 lines 1-2)."""
    import paper_1810_03063_b200 as P
    pair = Pair(kind="leduc", n_games=1)
    G = pair.game
    G.cfr_init(P.CFR_PLUS)
    G.cfr_step(3)
    states = []
    for _ in range(2):
        G.egt_init(P.EGT_AS)
        xs, ys = _strategies(G)
        states.append((G.egt_scalars()[:, :3].copy(), xs, ys))
    fresh = Pair(kind="leduc", n_games=1).game
    fresh.egt_init(P.EGT_AS)
    fx, fy = _strategies(fresh)
    for sc, xs, ys in states:
        assert np.array_equal(sc, fresh.egt_scalars()[:, :3])
        assert np.array_equal(xs, fx) and np.array_equal(ys, fy)
    k, mu = egt.practical_mu(pair.sf[0])
    prob = egt.Problem(pair.sf[0])
    x0, y0 = egt.initialize(prob, mu, mu)
    assert_scalar(states[0][0][0, 0], mu, 1e-14, "re-init practical mu", floor=0)
    assert_parity(pair.from_product(0, 0, fx[0])[1:], x0[1:], TOL, "re-init x0")
    assert_parity(pair.from_product(0, 1, fy[0])[1:], y0[1:], TOL, "re-init y0")
