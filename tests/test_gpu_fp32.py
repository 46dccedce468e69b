"""Row 9: the optional fp32 mode (fp32 vectors and arithmetic) against the fp64 oracle.

Bar (BASELINE.json north_star): relative error <= 1e-5 per element (paritylib.assert_parity,
absolute floor 1e-7 * max|oracle| for entries that cancel), per-game values relative.  Solvers are compared on
variants without an accept/reject decision (EGT with mu balancing, CFR+ on games without exact
regret ties), so fp32 rounding cannot flip a discrete choice (R18)."""
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


def test_cfr_plus_fp32(pair):
    if pair.kind == "kuhn" or pair.game.H > 1000:
        # Kuhn's exact regret ties, and the Libratus-scale game's hands with zero or tiny
        # regrets, make RM+'s [r]^+ switch on fp32 rounding noise (R18)
        pytest.skip("regret-matching decisions at the fp32 noise level")
    import paper_1810_03063_b200 as P
    G = pair.game
    G.cfr_init(P.CFR_PLUS)
    G.cfr_step(5)
    avg = _strategies(pair, 1)
    for g in range(G.n_games):
        st = cfr.run(pair.sf[g], "cfr_plus", 5)
        assert_parity(avg[0][g][1:], st.xbar[1:], TOL, "fp32 cfr+ xbar")
        assert_parity(avg[1][g][1:], st.ybar[1:], TOL, "fp32 cfr+ ybar")
