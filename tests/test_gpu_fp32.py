"""Row 9: the optional fp32 mode (fp32 vectors and arithmetic) against the fp64 oracle.

Bar (BASELINE.json north_star): relative error <= 1e-5 per element (paritylib.assert_parity,
absolute floor 1e-6 * max|oracle| for entries that cancel), per-game values relative.  Discrete
decisions taken on floating-point values (RM+'s [r]^+, EGT/as's EGV >= 0) are compared where
the oracle's fp64 margin exceeds the fp32 noise; a decision at the noise level may go either
way (R18) and what depends on it is left out -- no test is skipped."""
import numpy as np
import pytest

from oracle import br, cfr, dgf, egt
from paper_1810_03063_b200 import workloads
from tests.paritylib import Pair, assert_parity, assert_scalar, random_behavioral

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-5

CASES = {
    "kuhn": dict(kind="kuhn", n_games=2),
    "leduc": dict(kind="leduc", n_games=2),
    "river_tiny": dict(kind="river", n_games=3, seed=1),
    "libratus": dict(kind="river", n_games=2, seed=4, spec=workloads.river_spec("libratus"), build_sparse=False),
}


class Pair32(Pair):
    def __init__(self, **kw):
        import paper_1810_03063_b200 as P
        orig = P.Game

        def game32(*a, **k):
            k["precision"] = "f32"
            return orig(*a, **k)
        P.Game = game32
        try:
            super().__init__(**kw)
        finally:
            P.Game = orig


@pytest.fixture(scope="module", params=list(CASES))
def pair(request):
    return Pair32(**CASES[request.param])


def dev32(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


def test_precision_flag(pair):
    assert pair.game.precision == "f32"


@pytest.mark.parametrize("p", [0, 1])
def test_gradient_fp32(pair, p):
    G = pair.game
    o = 1 - p
    rng = np.random.default_rng(10 + p)
    ins, wants = [], []
    for g in range(G.n_games):
        v = pair.tp(g, o).behavioral_to_sequence(random_behavioral(pair.tp(g, o), rng))
        ins.append(pair.to_product(g, o, v, row0=1.0))
        sf = pair.sf[g]
        wants.append(sf.Ay(v) if p == 0 else sf.ATx(v))
    din = dev32(np.stack(ins).reshape(G.vec_shape(o)))
    dout = torch.full(G.vec_shape(p), np.nan, dtype=torch.float32, device="cuda")
    G.egt_gradient(p, din, dout)
    out = host(dout).reshape(G.n_games, -1)
    for g in range(G.n_games):
        got = pair.from_product(g, p, out[g])
        got[0] = out[g][:G.H_pad].sum()
        assert_parity(got, wants[g], TOL, "fp32 gradient")


@pytest.mark.parametrize("p,gsign", [(0, 1.0), (1, -1.0)])
def test_sbr_prox_br_fp32(pair, p, gsign):
    G = pair.game
    rng = np.random.default_rng(20 + p)
    gs, mus, cbs, steps, wsbr, wprox, wbr = [], [], [], [], [], [], []
    for g in range(G.n_games):
        tp = pair.tp(g, p)
        v = rng.standard_normal(tp.n_seq) * 3.0
        blk = pair.to_product(g, p, v)
        blk[0] = v[0]
        gs.append(blk)
        mu = float(np.exp(rng.uniform(-1, 1)))
        mus.append(mu)
        lb = np.log(random_behavioral(tp, rng, spread=1.0))
        cbs.append(pair.to_product(g, p, lb))
        st = float(np.exp(rng.uniform(-1, 0.5)))
        steps.append(st)
        wsbr.append(dgf.smoothed_best_response(tp, gsign * v, mu))
        vp = v.copy()
        vp[0] = 0.0
        wprox.append(dgf.prox_mapping(tp, st * gsign * vp, lb_prev=lb))
        wbr.append(br.best_response(tp, gsign * v, "min")[0])
    dg = dev32(np.stack(gs).reshape(G.vec_shape(p)))
    dq = torch.zeros(G.vec_shape(p), dtype=torch.float32, device="cuda")
    val = torch.zeros(G.n_games, dtype=torch.float64, device="cuda")
    G.egt_smoothed_br(p, dg, gsign, torch.tensor(mus, dtype=torch.float64, device="cuda"), dq, None, val)
    q, vals = host(dq).reshape(G.n_games, -1), host(val)
    for g in range(G.n_games):
        assert_parity(pair.from_product(g, p, q[g])[1:], wsbr[g][0][1:], TOL, "fp32 sbr q")
        assert_scalar(vals[g], wsbr[g][1], TOL, "fp32 sbr value")
    dq.zero_()
    G.egt_prox(p, dg, gsign, torch.tensor(steps, dtype=torch.float64, device="cuda"),
               dev32(np.stack(cbs).reshape(G.vec_shape(p))), dq)
    q = host(dq).reshape(G.n_games, -1)
    for g in range(G.n_games):
        assert_parity(pair.from_product(g, p, q[g])[1:], wprox[g][1:], TOL, "fp32 prox q")
    G.egt_best_response(p, dg, gsign, val)
    vals = host(val)
    for g in range(G.n_games):
        assert_scalar(vals[g], wbr[g], TOL, "fp32 br value")


def _strategies(pair, which):
    G = pair.game
    out = []
    for p in (0, 1):
        d = torch.zeros(G.vec_shape(p), dtype=torch.float32, device="cuda")
        G.get_strategy_device(p, which, d)
        a = host(d).reshape(G.n_games, -1)
        out.append([pair.from_product(g, p, a[g]) for g in range(G.n_games)])
    return out


def test_egt_balanced_fp32(pair):
    import paper_1810_03063_b200 as P
    G = pair.game
    mu = 0.5 * egt.theory_mu(pair.sf[0])
    G.egt_init(P.EGT_BALANCED, mu, mu)
    G.egt_step(4)
    xs, ys = _strategies(pair, 0)
    gaps = G.saddle_gap(0)
    for g in range(G.n_games):
        sf = pair.sf[g]
        prob = egt.Problem(sf)
        x, y = egt.initialize(prob, mu, mu)
        st = egt.EGTState(x, y, mu, mu)
        for _ in range(4):
            egt.egt_iteration(prob, st, "balanced")
        assert_parity(xs[g][1:], st.x[1:], TOL, "fp32 egt balanced x")
        assert_parity(ys[g][1:], st.y[1:], TOL, "fp32 egt balanced y")
        want = br.saddle_gap(sf, st.x, st.y)
        assert_scalar(gaps[g], want, TOL, "fp32 egt balanced eps_sad")


def _subtree_mask(tp, simplexes):
    """Sequences of the given simplexes and of every simplex below them."""
    bad = np.zeros(tp.n_seq, dtype=bool)
    for k in range(tp.n_simplex):  # top-down: a parent's mark is set before its children's
        s, n, par = tp.start[k], tp.size[k], tp.parent[k]
        if k in simplexes or (par != 0 and bad[par]):
            bad[s:s + n] = True
    return bad


def _fp32_perturbed(sf, seed):
    """The same sequence form with every gradient perturbed at the fp32 mode's own accuracy:
    1e-5 * max|g| per (nonzero) entry, the norm-relative bar test_gradient_fp32 holds it to --
    to measure how far that alone moves the oracle (an equally valid fp32-accurate computation)."""
    import copy
    alt = copy.copy(sf)
    rng = np.random.default_rng(seed)

    def noisy(f):
        def h(v):
            r = f(v)
            return r + 1e-5 * np.abs(r).max() * rng.standard_normal(r.shape) * (r != 0)
        return h
    alt.Ay, alt.ATx = noisy(sf.Ay), noisy(sf.ATx)
    return alt


def test_cfr_plus_fp32(pair):
    """Decision-aware (R18).  RM+'s "[r]^+ / r = 0" decisions taken within 1e-4 of the
    player's largest gain from flipping (traced from the fp64 oracle; fp32 gains are accurate to
    ~1e-5 of it) may go the other way in fp32: those simplexes and everything below them are left
    out, every other entry of both averages must match at 1e-5 per element -- plus 10x the
    oracle's own spread when its gradients are perturbed at the fp32 gradient's accuracy
    (1e-5 * max|g|): on the Libratus-scale game the regret decisions of low-prior hands cascade,
    and that perturbation alone moves CFR+'s 5-iteration averages by up to ~1e-1 and eps_sad by
    ~1e-4 -- and so must eps_sad."""
    import paper_1810_03063_b200 as P
    G = pair.game
    T = 5
    G.cfr_init(P.CFR_PLUS)
    G.cfr_step(T)
    avg = _strategies(pair, 1)
    gaps = G.saddle_gap(1)
    compared = total = 0
    for g in range(G.n_games):
        calls = []
        st = cfr.run(pair.sf[g], "cfr_plus", T, trace=lambda p, j, m, sj: calls.append((p, j, m, sj)))
        alt = cfr.run(_fp32_perturbed(pair.sf[g], 50 + g), "cfr_plus", T)
        # fp32 gains carry ~1e-5 of the largest gain of the pass (the norm-relative bar): a
        # regret within 1e-4 of that from the threshold may be decided the other way
        scale = [max([c[3] for c in calls if c[0] == p] or [0.0]) for p in (0, 1)]
        noisy = (set(), set())
        for p, j, m, sj in calls:
            if m <= 1e-4 * scale[p]:
                noisy[p].add(j)
        for p, want, other in ((0, st.xbar, alt.xbar), (1, st.ybar, alt.ybar)):
            keep = ~_subtree_mask(pair.tp(g, p), noisy[p])
            keep[0] = False
            spread = float(np.abs(other - want)[keep].max()) if keep.any() else 0.0
            assert_parity(avg[p][g][keep], want[keep], TOL, "fp32 cfr+ average (decided entries)",
                          floor=1e-5 + 10.0 * spread / max(np.abs(want).max(), 1e-300))
            compared += int(keep.sum())
            total += len(want) - 1
        want_gap = br.saddle_gap(pair.sf[g], st.xbar, st.ybar)
        spread_gap = abs(br.saddle_gap(pair.sf[g], alt.xbar, alt.ybar) - want_gap)
        assert_scalar(gaps[g], want_gap, TOL, "fp32 cfr+ eps_sad", floor=10.0 * spread_gap)
    # (exact regret ties -- Kuhn, Leduc -- and low-prior hands leave many entries out)
    assert compared >= 0.1 * total, (compared, total)
    print("fp32 cfr+ [%s]: %d of %d average entries compared" % (pair.kind, compared, total))


def test_egt_as_fp32(pair):
    """EGT/as (Alg. 3-4) in fp32 against the fp64 oracle, attempt by attempt: the accept /
    backtrack decision (EGV >= 0) must match wherever the oracle's EGV is further than 1e-4 of
    its scale (|phi| + |f|) from 0 (R18); up to the first decision at that noise
    level, mu, tau, the iterate and eps_sad match at 1e-5."""
    import paper_1810_03063_b200 as P
    G = pair.game
    mu = egt.theory_mu(pair.sf[0]) / 8.0
    G.egt_init(P.EGT_AS, mu, mu)
    states = []
    for g in range(G.n_games):
        prob = egt.Problem(pair.sf[g])
        x, y = egt.initialize(prob, mu, mu)
        states.append((prob, egt.EGTState(x, y, mu, mu), [True]))
    n_decisions = 0
    for attempt in range(8):
        G.egt_step(1)
        sc = G.egt_scalars()
        xs, ys = _strategies(pair, 0)
        gaps = G.saddle_gap(0)
        for g, (prob, st, live) in enumerate(states):
            if not live[0]:
                continue
            focus = "x" if st.mu_x > st.mu_y else "y"
            mx, my, xn, yn = egt.step_xy(prob, st, focus, st.tau)
            phi, _ = egt.smoothed_phi(prob, yn, mx)
            f, _ = egt.smoothed_f(prob, xn, my)
            accept = phi - f >= 0
            if accept:
                st.mu_x, st.mu_y, st.x, st.y = mx, my, xn, yn
                st.t += 1
            else:
                st.tau *= 0.5
                st.backtracks += 1
            if int(sc[g, 3]) != st.t or int(sc[g, 5]) != st.backtracks:
                assert abs(phi - f) <= 1e-4 * (abs(phi) + abs(f)), ("decision off the noise level", g, attempt)
                live[0] = False  # a noise-level decision went the other way: stop comparing this game
                continue
            n_decisions += 1
            assert_scalar(sc[g, 0], st.mu_x, TOL, "fp32 egt/as mu", floor=0)
            assert_scalar(sc[g, 1], st.mu_y, TOL, "fp32 egt/as mu", floor=0)
            assert_scalar(sc[g, 2], st.tau, TOL, "fp32 egt/as tau", floor=0)
            assert_parity(xs[g][1:], st.x[1:], TOL, "fp32 egt/as x")
            assert_parity(ys[g][1:], st.y[1:], TOL, "fp32 egt/as y")
            assert_scalar(gaps[g], br.saddle_gap(pair.sf[g], st.x, st.y), TOL, "fp32 egt/as eps_sad")
    assert n_decisions >= 4 * G.n_games
