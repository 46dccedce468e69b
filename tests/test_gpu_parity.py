"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element by element.

Tolerance: fp64 end to end; every element of a vector
result within 1e-9 relative of the oracle's, with an absolute floor of 1e-13 * max|oracle|
for entries that cancel to ~0 (paritylib.assert_parity); per-game values and eps_sad 1e-9
relative.  Integer/index work (layout) is compared exactly.
"""
import numpy as np
import pytest

from oracle import br, cfr, dgf, egt
from tests.paritylib import Pair, assert_parity, assert_scalar, random_behavioral

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-9

CASES = {
    "kuhn": dict(kind="kuhn", n_games=2),
    "leduc": dict(kind="leduc", n_games=2),
    "river_tiny": dict(kind="river", n_games=3, seed=1),
}


@pytest.fixture(scope="module", params=list(CASES))
def pair(request):
    return Pair(**CASES[request.param])


def dev(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def stack(pair, p, blocks):
    G = pair.game
    return np.stack(blocks).reshape(G.n_games, G.n_pub[p], G.H_pad)


# ------------------------------------------------------------------ layout (exact)
def test_layout_bijection(pair):
    G = pair.game
    for g in range(G.n_games):
        for p in (0, 1):
            idx = pair.index_map(g, p)
            assert len(np.unique(idx)) == len(idx) == pair.tp(g, p).n_seq - 1
            assert (idx % G.H_pad < G.H).all()


# ------------------------------------------------------------------ gradient
@pytest.mark.parametrize("p", [0, 1])
def test_gradient(pair, p):
    G = pair.game
    o = 1 - p
    rng = np.random.default_rng(10 + p)
    ins, wants = [], []
    for g in range(G.n_games):
        v = pair.tp(g, o).behavioral_to_sequence(random_behavioral(pair.tp(g, o), rng))
        ins.append(pair.to_product(g, o, v, row0=1.0))
        sf = pair.sf[g]
        wants.append(sf.Ay(v) if p == 0 else sf.ATx(v))
    din = dev(stack(pair, o, ins))
    dout = torch.full((G.n_games,) + G.vec_shape(p)[1:], np.nan, dtype=torch.float64, device="cuda")
    G.egt_gradient(p, din, dout)
    out = host(dout).reshape(G.n_games, -1)
    for g in range(G.n_games):
        got = pair.from_product(g, p, out[g])
        got[0] = out[g][:G.H_pad].sum()
        assert_parity(got, wants[g], TOL, "gradient[%s]" % pair.kind)
        invalid = ~pair.valid_mask(g, p)
        invalid[:G.H_pad] = False
        assert np.all(out[g][invalid] == 0.0)


# ------------------------------------------------------------------ smoothed best response
@pytest.mark.parametrize("p,gsign", [(0, 1.0), (1, -1.0), (1, 1.0)])
def test_smoothed_best_response(pair, p, gsign):
    G = pair.game
    rng = np.random.default_rng(20 + p)
    gs, mus, wants = [], [], []
    for g in range(G.n_games):
        tp = pair.tp(g, p)
        v = rng.standard_normal(tp.n_seq) * 3.0
        mu = float(np.exp(rng.uniform(-2, 1)))
        blk = pair.to_product(g, p, v)
        blk[0] = v[0]  # empty-sequence term on one hand column
        gs.append(blk)
        mus.append(mu)
        wants.append(dgf.smoothed_best_response(tp, gsign * v, mu, behavioral=True))
    dq = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
    db = torch.zeros_like(dq)
    val = torch.zeros(G.n_games, dtype=torch.float64, device="cuda")
    dlb = torch.zeros_like(dq)
    G.egt_smoothed_br(p, dev(stack(pair, p, gs)), gsign, dev(mus), dq, db, val, lb=dlb)
    q = host(dq).reshape(G.n_games, -1)
    b = host(db).reshape(G.n_games, -1)
    lb = host(dlb).reshape(G.n_games, -1)
    vals = host(val)
    for g in range(G.n_games):
        wq, wv, wb, wlb = wants[g]
        assert_parity(pair.from_product(g, p, q[g])[1:], wq[1:], TOL, "sbr q[%s]" % pair.kind)
        assert_parity(pair.from_product(g, p, b[g])[1:], wb[1:], TOL, "sbr b[%s]" % pair.kind)
        assert_parity(pair.from_product(g, p, lb[g])[1:], wlb[1:], TOL, "sbr log b[%s]" % pair.kind)
        assert_scalar(vals[g], wv, TOL, "sbr value[%s]" % pair.kind)


# ------------------------------------------------------------------ prox mapping
@pytest.mark.parametrize("p,gsign,far", [(0, 1.0, False), (1, -1.0, False), (0, 1.0, True), (1, -1.0, True)])
def test_prox(pair, p, gsign, far):
    """Centres given by their behavioural logs (R16); `far`: entries at log ~ -800
    (underflowing probabilities, the practical-mu regime) pulled back by large gradients."""
    G = pair.game
    rng = np.random.default_rng(30 + p)
    gs, steps, cbs, wants = [], [], [], []
    for g in range(G.n_games):
        tp = pair.tp(g, p)
        v = rng.standard_normal(tp.n_seq)
        s = float(np.exp(rng.uniform(-2, 1)))
        lb = np.log(random_behavioral(tp, rng, spread=1.5))
        if far:  # centres at the bench's operating point: behavioural probabilities ~e^-800
            for j in range(tp.n_simplex):
                st_, n_ = tp.start[j], tp.size[j]
                t = lb[st_:st_ + n_].copy()
                keep = int(np.argmax(t))
                for i in range(n_):
                    if i != keep and rng.random() < 0.4:
                        t[i] -= 800.0
                        if rng.random() < 0.7:  # and a gradient that pulls it back into play
                            v[st_ + i] = 0.99 * t[i] * tp.beta[j] / (s * gsign)
                m = t.max()
                lb[st_:st_ + n_] = t - (m + np.log(np.exp(t - m).sum()))
        gs.append(pair.to_product(g, p, v))
        steps.append(s)
        cbs.append(pair.to_product(g, p, lb))
        wants.append(dgf.prox_mapping(tp, s * gsign * v, lb_prev=lb))
    dq = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
    G.egt_prox(p, dev(stack(pair, p, gs)), gsign, dev(steps), dev(stack(pair, p, cbs)), dq)
    q = host(dq).reshape(G.n_games, -1)
    for g in range(G.n_games):
        assert_parity(pair.from_product(g, p, q[g])[1:], wants[g][1:], TOL, "prox[%s]" % pair.kind)


# ------------------------------------------------------------------ best response
@pytest.mark.parametrize("p", [0, 1])
def test_best_response(pair, p):
    G = pair.game
    rng = np.random.default_rng(40 + p)
    gs, wants = [], []
    for g in range(G.n_games):
        tp = pair.tp(g, p)
        v = rng.standard_normal(tp.n_seq)
        blk = pair.to_product(g, p, v)
        blk[0] = v[0]
        gs.append(blk)
        wants.append((br.best_response(tp, v, "min")[0], br.best_response(tp, -v, "min")[0]))
    val = torch.zeros(G.n_games, dtype=torch.float64, device="cuda")
    for k, gsign in enumerate((1.0, -1.0)):
        G.egt_best_response(p, dev(stack(pair, p, gs)), gsign, val)
        got = host(val)
        for g in range(G.n_games):
            assert_scalar(got[g], wants[g][k], TOL, "br value[%s]" % pair.kind)


# ------------------------------------------------------------------ solvers
def _strategies(pair, which=1):
    G = pair.game
    out = []
    for p in (0, 1):
        d = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        G.get_strategy_device(p, which, d)
        a = host(d).reshape(G.n_games, -1)
        out.append([pair.from_product(g, p, a[g]) for g in range(G.n_games)])
    return out


@pytest.mark.parametrize("variant,iters", [("theory", 6), ("balanced", 8), ("as", 10)])
def test_egt_iterates(pair, variant, iters):
    import paper_1810_03063_b200 as P
    G = pair.game
    code = {"theory": P.EGT_THEORY, "balanced": P.EGT_BALANCED, "as": P.EGT_AS}[variant]
    sf0 = pair.sf[0]
    mu = 0.5 * egt.theory_mu(sf0) if variant != "theory" else None
    if variant == "theory":
        G.egt_init(code)
    else:
        G.egt_init(code, mu, mu)
    sc0 = G.egt_scalars()
    G.egt_step(iters)
    sc = G.egt_scalars()
    x_all, y_all = _strategies(pair, 0)
    gaps = G.saddle_gap(0)
    for g in range(G.n_games):
        sf = pair.sf[g]
        prob = egt.Problem(sf)
        m = egt.theory_mu(sf) if variant == "theory" else mu
        if variant == "theory":
            assert abs(sc0[g, 0] - m) <= TOL * m and abs(sc0[g, 1] - m) <= TOL * m
        x, y = egt.initialize(prob, m, m)
        st = egt.EGTState(x, y, m, m)
        accepted = int(sc[g, 3])
        for _ in range(accepted):
            egt.egt_iteration(prob, st, variant)
        if variant == "as":
            assert int(sc[g, 4]) == iters and accepted + int(sc[g, 5]) == iters
            assert st.backtracks == int(sc[g, 5])
        else:
            assert accepted == iters
        assert_parity(x_all[g][1:], st.x[1:], TOL, "egt x[%s]" % pair.kind)
        assert_parity(y_all[g][1:], st.y[1:], TOL, "egt y[%s]" % pair.kind)
        assert_scalar(sc[g, 0], st.mu_x, TOL, "egt mu", floor=0)
        assert_scalar(sc[g, 1], st.mu_y, TOL, "egt mu", floor=0)
        if variant == "as":  # theory / balanced use tau_t = 2/(t+3), not the EGT/as state's tau
            assert_scalar(sc[g, 2], st.tau, TOL, "egt tau", floor=0)
        want_gap = br.saddle_gap(sf, st.x, st.y)
        assert_scalar(gaps[g], want_gap, TOL, "egt eps_sad[%s]" % pair.kind)


@pytest.mark.parametrize("variant", ["cfr_rm", "cfr_rmp", "cfr_plus"])
def test_cfr_iterates(pair, variant):
    import paper_1810_03063_b200 as P
    G = pair.game
    code = {"cfr_rm": P.CFR_RM, "cfr_rmp": P.CFR_RMP, "cfr_plus": P.CFR_PLUS}[variant]
    iters = 12
    G.cfr_init(code)
    G.cfr_step(iters)
    cur = _strategies(pair, 0)
    avg = _strategies(pair, 1)
    gaps = G.saddle_gap(1)
    for g in range(G.n_games):
        st = cfr.run(pair.sf[g], variant, iters)
        assert_parity(cur[0][g][1:], st.x[1:], TOL, "cfr x[%s]" % pair.kind)
        assert_parity(cur[1][g][1:], st.y[1:], TOL, "cfr y[%s]" % pair.kind)
        assert_parity(avg[0][g][1:], st.xbar[1:], TOL, "cfr xbar[%s]" % pair.kind)
        assert_parity(avg[1][g][1:], st.ybar[1:], TOL, "cfr ybar[%s]" % pair.kind)
        want = br.saddle_gap(pair.sf[g], st.xbar, st.ybar)
        assert_scalar(gaps[g], want, TOL, "cfr eps_sad[%s]" % pair.kind)


def test_avg_strategy_canonical_layout(pair):
    """get_avg_strategy (HOST, canonical combo order) agrees with the device layout."""
    import paper_1810_03063_b200 as P
    G = pair.game
    G.cfr_init(P.CFR_PLUS)
    G.cfr_step(3)
    avg = _strategies(pair, 1)
    for p in (0, 1):
        hostv = G.get_avg_strategy(p)
        assert hostv.shape == (G.n_games, G.n_pub[p], G.n_combos)
        for g in range(G.n_games):
            cards = G.hand_cards(g)
            for h in range(min(G.H, 7)):
                c = [x for x in cards[h] if x >= 0]
                combo = c[0] if len(c) == 1 else _combo_index(c[0], c[1], _n_cards(pair))
                for s in range(1, G.n_pub[p]):
                    flat = s * G.H_pad + h
                    i = np.where(pair.index_map(g, p) == flat)[0]
                    want = avg[p][g][1 + i[0]] if len(i) else 0.0
                    assert hostv[g, s, combo] == want


def _n_cards(pair):
    return {"kuhn": 3, "leduc": 6}.get(pair.kind, 52)


def _combo_index(c1, c2, n):
    return c1 * (2 * n - c1 - 1) // 2 + (c2 - c1 - 1)


def test_card_domain_kernel_parity():
    """The card-domain gradient kernel (EGT_GRAD_KERNEL=card; the library launches the staged
    one by default) against the oracle, in a process of its own (the switch is read once)."""
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, torch
from paper_1810_03063_b200 import workloads
from tests.paritylib import Pair, assert_parity, random_behavioral
for spec, seed, nr, ns in ((workloads.river_spec("libratus"), 4, 13, 4), (workloads.river_spec("simple"), 9, 8, 4)):
    pair = Pair("river", n_games=2, spec=spec, seed=seed, n_ranks=nr, n_suits=ns, build_sparse=False)
    G = pair.game
    rng = np.random.default_rng(1)
    for p in (0, 1):
        o = 1 - p
        blocks, vals = [], []
        for g in range(G.n_games):
            v = pair.tp(g, o).behavioral_to_sequence(random_behavioral(pair.tp(g, o), rng))
            vals.append(v)
            blocks.append(pair.to_product(g, o, v, row0=1.0))
        din = torch.tensor(np.stack(blocks).reshape(G.vec_shape(o)), device="cuda")
        dout = torch.full(G.vec_shape(p), np.nan, dtype=torch.float64, device="cuda")
        G.egt_gradient(p, din, dout)
        torch.cuda.synchronize()
        out = dout.cpu().numpy().reshape(G.n_games, -1)
        for g in range(G.n_games):
            want = pair.sf[g].Ay(vals[g]) if p == 0 else pair.sf[g].ATx(vals[g])
            got = pair.from_product(g, p, out[g])
            got[0] = out[g][:G.H_pad].sum()
            assert_parity(got, want, 1e-9, "card-domain gradient")
print("card kernel ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, EGT_GRAD_KERNEL="card", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "card kernel ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
