"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The bench workload (296 Libratus-scale endgames per GPU: the paper's full bet abstraction,
1081 hands, 153 public sequences per player, 203 terminals) goes through the C ABI exactly as
bench.py builds it; the oracle (``oracle/``) recomputes sampled games one by one.  Edge cases:
a board on which every hand ties, very sparse priors, a single-hand range, and reduced decks
whose hand count leaves a ragged tail in the 32-hand tiles.
"""
import numpy as np
import pytest

from oracle import br, cfr, dgf, egt
from paper_1810_03063_b200 import workloads
from tests.paritylib import Pair, assert_parity, assert_scalar, random_behavioral

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-9
BENCH_BATCH = 296
SAMPLE = (0, 147, 295)


def dev(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def bench_pair():
    import bench
    args = type("A", (), {"workload": "libratus", "seed": 2100, "batch": BENCH_BATCH})()
    spec, boards, p1, p2 = bench.workload(args, 0)
    return Pair("river", n_games=BENCH_BATCH, spec=spec, boards=boards, priors=(p1, p2), sample=SAMPLE,
                build_sparse=False)


def _full_inputs(pair, p, rng, games):
    """Random behavioural strategies of player p (sampled games), zeros elsewhere (row 0 = 1)."""
    G = pair.game
    blocks = np.zeros((G.n_games, G.n_pub[p] * G.H_pad))
    blocks[:, :G.H] = 1.0
    vals = {}
    for g in games:
        v = pair.tp(g, p).behavioral_to_sequence(random_behavioral(pair.tp(g, p), rng))
        vals[g] = v
        blocks[g] = pair.to_product(g, p, v, row0=1.0)
    return blocks.reshape((G.n_games,) + G.vec_shape(p)[1:]), vals


@pytest.mark.parametrize("p", [0, 1])
def test_bench_workload_gradient(bench_pair, p):
    pair, G = bench_pair, bench_pair.game
    assert (G.H, G.n_pub, G.n_terminals) == (1081, (153, 153), 203)
    o = 1 - p
    blocks, vals = _full_inputs(pair, o, np.random.default_rng(100 + p), SAMPLE)
    dout = torch.full((G.n_games,) + G.vec_shape(p)[1:], np.nan, dtype=torch.float64, device="cuda")
    G.egt_gradient(p, dev(blocks), dout)
    out = host(dout).reshape(G.n_games, -1)
    assert np.isfinite(out).all()
    for g in SAMPLE:
        sf = pair.sf[g]
        want = sf.Ay(vals[g]) if p == 0 else sf.ATx(vals[g])
        got = pair.from_product(g, p, out[g])
        got[0] = out[g][:G.H_pad].sum()
        assert_parity(got, want, TOL, "bench-batch gradient")


def test_bench_workload_sbr_and_br(bench_pair):
    pair, G = bench_pair, bench_pair.game
    rng = np.random.default_rng(7)
    for p, gsign in ((0, 1.0), (1, -1.0)):
        gs = np.zeros((G.n_games, G.n_pub[p] * G.H_pad))
        mus = np.ones(G.n_games)
        wants = {}
        for g in SAMPLE:
            v = rng.standard_normal(pair.tp(g, p).n_seq) * 50.0
            gs[g] = pair.to_product(g, p, v)
            gs[g][0] = v[0]
            mus[g] = float(np.exp(rng.uniform(-1, 3)))
            wants[g] = (dgf.smoothed_best_response(pair.tp(g, p), gsign * v, mus[g]),
                        br.best_response(pair.tp(g, p), gsign * v, "min")[0])
        dg = dev(gs.reshape((G.n_games,) + G.vec_shape(p)[1:]))
        dq = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        val = torch.zeros(G.n_games, dtype=torch.float64, device="cuda")
        bval = torch.zeros_like(val)
        G.egt_smoothed_br(p, dg, gsign, dev(mus), dq, None, val)
        G.egt_best_response(p, dg, gsign, bval)
        q, vals, bvals = host(dq).reshape(G.n_games, -1), host(val), host(bval)
        for g in SAMPLE:
            (wq, wv), wb = wants[g]
            assert_parity(pair.from_product(g, p, q[g])[1:], wq[1:], TOL, "bench-batch sbr q")
            assert_scalar(vals[g], wv, TOL, "bench-batch sbr value")
            assert_scalar(bvals[g], wb, TOL, "bench-batch br value")


def test_bench_workload_egt_as_iterations(bench_pair):
    """EGT/as on the whole bench batch (graph-launched steps), game 0 against the oracle."""
    import paper_1810_03063_b200 as P
    pair, G = bench_pair, bench_pair.game
    g = SAMPLE[0]
    sf = pair.sf[g]
    mu = egt.theory_mu(sf) * 2.0 ** -6
    G.egt_init(P.EGT_AS, mu, mu)
    G.egt_step(2)
    sc = G.egt_scalars()
    xs = torch.zeros(G.vec_shape(0), dtype=torch.float64, device="cuda")
    ys = torch.zeros(G.vec_shape(1), dtype=torch.float64, device="cuda")
    G.get_strategy_device(0, 0, xs)
    G.get_strategy_device(1, 0, ys)
    gaps = G.saddle_gap(0)
    prob = egt.Problem(sf)
    x, y = egt.initialize(prob, mu, mu)
    st = egt.EGTState(x, y, mu, mu)
    for _ in range(int(sc[g, 3])):
        egt.egt_iteration(prob, st, "as")
    assert int(sc[g, 3]) + int(sc[g, 5]) == 2 and st.backtracks == int(sc[g, 5])
    assert_parity(pair.from_product(g, 0, host(xs).reshape(G.n_games, -1)[g])[1:], st.x[1:], TOL, "bench-batch egt/as x")
    assert_parity(pair.from_product(g, 1, host(ys).reshape(G.n_games, -1)[g])[1:], st.y[1:], TOL, "bench-batch egt/as y")
    want = br.saddle_gap(sf, st.x, st.y)
    assert_scalar(gaps[g], want, TOL, "bench-batch egt/as eps_sad")
    assert np.all(gaps >= -1e-9 * np.abs(gaps).max())


def test_bench_workload_cfr_plus(bench_pair):
    import paper_1810_03063_b200 as P
    pair, G = bench_pair, bench_pair.game
    g = SAMPLE[-1]
    G.cfr_init(P.CFR_PLUS)
    G.cfr_step(2)
    avg = []
    for p in (0, 1):
        d = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        G.get_strategy_device(p, 1, d)
        avg.append(pair.from_product(g, p, host(d).reshape(G.n_games, -1)[g]))
    gaps = G.saddle_gap(1)
    st = cfr.run(pair.sf[g], "cfr_plus", 2)
    assert_parity(avg[0][1:], st.xbar[1:], TOL, "bench-batch cfr+ xbar")
    assert_parity(avg[1][1:], st.ybar[1:], TOL, "bench-batch cfr+ ybar")
    want = br.saddle_gap(pair.sf[g], st.xbar, st.ybar)
    assert_scalar(gaps[g], want, TOL, "bench-batch cfr+ eps_sad")


# ------------------------------------------------------------------ edge cases
def _gradient_parity(pair, games=None):
    G = pair.game
    games = list(range(G.n_games)) if games is None else games
    for p in (0, 1):
        o = 1 - p
        blocks, vals = _full_inputs(pair, o, np.random.default_rng(5 + p), games)
        dout = torch.full((G.n_games,) + G.vec_shape(p)[1:], np.nan, dtype=torch.float64, device="cuda")
        G.egt_gradient(p, dev(blocks), dout)
        out = host(dout).reshape(G.n_games, -1)
        for g in games:
            sf = pair.sf[g]
            want = sf.Ay(vals[g]) if p == 0 else sf.ATx(vals[g])
            got = pair.from_product(g, p, out[g])
            got[0] = out[g][:G.H_pad].sum()
            assert_parity(got, want, TOL, "edge-case gradient")
            assert np.all(out[g][G.H:G.H_pad] == 0.0)


def test_all_hands_tie_board():
    """Royal-flush board: every hand plays the board, every showdown is a split pot."""
    # card id = rank_pos * 4 + suit, rank_pos 12 = ace: A K Q J T of suit 0
    boards = np.array([[48, 44, 40, 36, 32], [0, 5, 22, 39, 51]], dtype=np.int32)
    pr = workloads.random_priors(boards, 11)
    pair = Pair("river", n_games=2, spec=workloads.river_spec("libratus"), boards=boards, priors=pr,
                build_sparse=False)
    _gradient_parity(pair)


def test_sparse_and_single_hand_priors():
    boards = workloads.random_boards(3, 21)
    p1, p2 = workloads.random_priors(boards, 21, zero_frac=0.97)
    # game 2: player 1 holds exactly one hand
    nz = np.flatnonzero(p1[2])
    keep = nz[len(nz) // 2]
    p1[2] = 0.0
    p1[2, keep] = 1.0
    pair = Pair("river", n_games=3, spec=workloads.river_spec("simple"), boards=boards, priors=(p1, p2),
                build_sparse=False)
    _gradient_parity(pair)


@pytest.mark.parametrize("n_ranks,n_suits", [(8, 4), (6, 3), (13, 2)])
def test_reduced_decks_ragged_tiles(n_ranks, n_suits):
    """Hand counts that are not multiples of 32 (351, 78, 190): ragged tails everywhere."""
    pair = Pair("river", n_games=2, spec=workloads.river_spec("simple"), seed=9, n_ranks=n_ranks, n_suits=n_suits,
                build_sparse=False)
    G = pair.game
    assert G.H % 32 != 0
    _gradient_parity(pair)
    rng = np.random.default_rng(3)
    for p, gsign in ((0, 1.0), (1, -1.0)):
        gs, mus, wants = [], [], []
        for g in range(G.n_games):
            v = rng.standard_normal(pair.tp(g, p).n_seq) * 5.0
            blk = pair.to_product(g, p, v)
            blk[0] = v[0]
            gs.append(blk)
            mus.append(0.7)
            wants.append(dgf.smoothed_best_response(pair.tp(g, p), gsign * v, 0.7))
        dq = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        val = torch.zeros(G.n_games, dtype=torch.float64, device="cuda")
        G.egt_smoothed_br(p, dev(np.stack(gs).reshape(G.vec_shape(p))), gsign, dev(mus), dq, None, val)
        q, vals = host(dq).reshape(G.n_games, -1), host(val)
        for g in range(G.n_games):
            assert_parity(pair.from_product(g, p, q[g])[1:], wants[g][0][1:], TOL, "edge-case sbr q")
            assert_scalar(vals[g], wants[g][1], TOL, "edge-case sbr value")


@pytest.mark.parametrize("variant", ["cfr_rm", "cfr_rmp"])
def test_bench_workload_cfr_variants(bench_pair, variant):
    """CFR(RM) and CFR(RM+) (uniform averaging) on the whole bench batch, one sampled game
    against the oracle: averages and their saddle-point gap after 2 iterations."""
    import paper_1810_03063_b200 as P
    pair, G = bench_pair, bench_pair.game
    g = SAMPLE[1]
    G.cfr_init({"cfr_rm": P.CFR_RM, "cfr_rmp": P.CFR_RMP}[variant])
    G.cfr_step(2)
    avg = []
    for p in (0, 1):
        d = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        G.get_strategy_device(p, 1, d)
        avg.append(pair.from_product(g, p, host(d).reshape(G.n_games, -1)[g]))
    gaps = G.saddle_gap(1)
    st = cfr.run(pair.sf[g], variant, 2)
    assert_parity(avg[0][1:], st.xbar[1:], TOL, "bench-batch cfr avg x")
    assert_parity(avg[1][1:], st.ybar[1:], TOL, "bench-batch cfr avg y")
    want = br.saddle_gap(pair.sf[g], st.xbar, st.ybar)
    assert_scalar(gaps[g], want, TOL, "bench-batch cfr eps_sad")


def test_bench_workload_egt_balanced(bench_pair):
    """EGT with mu balancing on the whole bench batch: game 295's iterate
    after 2 graph-launched iterations against the oracle."""
    import paper_1810_03063_b200 as P
    pair, G = bench_pair, bench_pair.game
    g = SAMPLE[-1]
    sf = pair.sf[g]
    mu = egt.theory_mu(sf) * 2.0 ** -4
    G.egt_init(P.EGT_BALANCED, mu, mu)
    G.egt_step(2)
    xs = torch.zeros(G.vec_shape(0), dtype=torch.float64, device="cuda")
    ys = torch.zeros(G.vec_shape(1), dtype=torch.float64, device="cuda")
    G.get_strategy_device(0, 0, xs)
    G.get_strategy_device(1, 0, ys)
    st, prob = egt.run(sf, "balanced", 2, mu=mu)
    assert_parity(pair.from_product(g, 0, host(xs).reshape(G.n_games, -1)[g])[1:], st.x[1:], TOL, "bench-batch egt balanced x")
    assert_parity(pair.from_product(g, 1, host(ys).reshape(G.n_games, -1)[g])[1:], st.y[1:], TOL, "bench-batch egt balanced y")
    gaps = G.saddle_gap(0)
    want = br.saddle_gap(sf, st.x, st.y)
    assert_scalar(gaps[g], want, TOL, "bench-batch egt balanced eps_sad")


@pytest.mark.parametrize("solver", ["egt_as", "cfr_plus"])
def test_bench_workload_longer_runs(bench_pair, solver):
    """Eight graph-launched iterations on the whole bench batch (EGT/as; CFR+), game 147
    against the oracle: iterate / average, counters, eps_sad.  EGT/as starts from mu_theory/16
    so that every prox centre stays interior for the oracle's literal prox form (DESIGN.md
    R16; the practical mu search drives smoothed responses to fp64 underflow within a few
    iterations, where only the kernel's multiplicative form is defined)."""
    import paper_1810_03063_b200 as P
    pair, G = bench_pair, bench_pair.game
    g = SAMPLE[1]
    sf = pair.sf[g]
    n = 8
    if solver == "egt_as":
        mu_x = mu_y = egt.theory_mu(sf) / 16.0
        G.egt_init(P.EGT_AS, mu_x, mu_y)
        G.egt_step(n)
        sc = G.egt_scalars()
        prob = egt.Problem(sf)
        x, y = egt.initialize(prob, mu_x, mu_y)
        st = egt.EGTState(x, y, mu_x, mu_y)
        for _ in range(int(sc[g, 3])):
            egt.egt_iteration(prob, st, "as")
        assert int(sc[g, 3]) + int(sc[g, 5]) == n and st.backtracks == int(sc[g, 5])
        assert abs(sc[g, 0] - st.mu_x) <= 1e-12 * st.mu_x and abs(sc[g, 1] - st.mu_y) <= 1e-12 * st.mu_y
        which, want_x, want_y = 0, st.x, st.y
    else:
        G.cfr_init(P.CFR_PLUS)
        G.cfr_step(n)
        st = cfr.run(sf, "cfr_plus", n)
        which, want_x, want_y = 1, st.xbar, st.ybar
    got = []
    for p in (0, 1):
        d = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        G.get_strategy_device(p, which, d)
        got.append(pair.from_product(g, p, host(d).reshape(G.n_games, -1)[g]))
    assert_parity(got[0][1:], want_x[1:], TOL, "bench-batch long-run x")
    assert_parity(got[1][1:], want_y[1:], TOL, "bench-batch long-run y")
    gaps = G.saddle_gap(which)
    want = br.saddle_gap(sf, want_x, want_y)
    assert_scalar(gaps[g], want, TOL, "bench-batch long-run eps_sad")


def _sweep_specs():
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import grad_sweep
    return grad_sweep.specs()


@pytest.mark.parametrize("which", range(5))
def test_sweep_abstractions_gradient(which):
    """BASELINE.json configs[4]'s five bet abstractions (tools/grad_sweep.py), from 18 to 348
    public sequences per player and 23 to 463 terminals -- the largest trees the gradient kernel
    is timed on, with the most terminals per chunk and the longest sequence indices -- on full
    52-card river boards with bench-style priors: both gradients per element against the oracle
    (Gen-CFR lines 29/35), then the smoothed best response and the best response
    on the same treeplexes."""
    name, spec = _sweep_specs()[which]
    boards = workloads.random_boards(4, seed=700 + which)
    priors = workloads.random_priors(boards, seed=700 + which)
    pair = Pair("river", n_games=4, spec=spec, boards=boards, priors=priors, sample=(0, 3), build_sparse=False)
    G = pair.game
    for p in (0, 1):
        blocks, vals = _full_inputs(pair, 1 - p, np.random.default_rng(710 + which + p), (0, 3))
        dout = torch.full((G.n_games,) + G.vec_shape(p)[1:], np.nan, dtype=torch.float64, device="cuda")
        G.egt_gradient(p, dev(blocks), dout)
        out = host(dout).reshape(G.n_games, -1)
        assert np.isfinite(out).all(), name
        for g in (0, 3):
            sf = pair.sf[g]
            want = sf.Ay(vals[g]) if p == 0 else sf.ATx(vals[g])
            got = pair.from_product(g, p, out[g])
            got[0] = out[g][:G.H_pad].sum()
            assert_parity(got, want, TOL, "sweep-abstraction gradient")
    # the treeplex passes on the same trees (nodes of up to 11 actions go through the
    # kernel's generic in-shared-memory path): smoothed best response and best response
    rng = np.random.default_rng(720 + which)
    for p, gsign in ((0, 1.0), (1, -1.0)):
        gs = np.zeros((G.n_games, G.n_pub[p] * G.H_pad))
        mus = np.ones(G.n_games)
        wants = {}
        for g in (0, 3):
            v = rng.standard_normal(pair.tp(g, p).n_seq) * 50.0
            gs[g] = pair.to_product(g, p, v)
            gs[g][0] = v[0]
            mus[g] = float(np.exp(rng.uniform(-1, 3)))
            wants[g] = (dgf.smoothed_best_response(pair.tp(g, p), gsign * v, mus[g]),
                        br.best_response(pair.tp(g, p), gsign * v, "min")[0])
        dg = dev(gs.reshape((G.n_games,) + G.vec_shape(p)[1:]))
        dq = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        val = torch.zeros(G.n_games, dtype=torch.float64, device="cuda")
        bval = torch.zeros_like(val)
        G.egt_smoothed_br(p, dg, gsign, dev(mus), dq, None, val)
        G.egt_best_response(p, dg, gsign, bval)
        q, vals, bvals = host(dq).reshape(G.n_games, -1), host(val), host(bval)
        for g in (0, 3):
            (wq, wv), wb = wants[g]
            assert_parity(pair.from_product(g, p, q[g])[1:], wq[1:], TOL, "sweep-abstraction sbr q")
            assert_scalar(vals[g], wv, TOL, "sweep-abstraction sbr value")
            assert_scalar(bvals[g], wb, TOL, "sweep-abstraction br value")
