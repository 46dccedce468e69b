"""Seeded random river configurations (decks, bet fractions, raise caps, open fold, all-in,
stacks) -- gradients of both players and one EGT/as iteration against the oracle.  Each case
is small enough for the oracle; together they reach code paths the fixed workloads do not
(lane-group widths other than 8, odd hand counts, few terminals per row, deep raise chains)."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import egt
from paper_1810_03063_b200 import workloads
from tests.paritylib import Pair, assert_parity, assert_scalar, random_behavioral

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-9
FRACS = ["1/4", "1/3", "1/2", "2/3", "3/4", "1", "3/2", "2"]


def random_spec(rng):
    spec = workloads.river_spec("tiny")
    spec["fracs"] = {k: sorted(set(rng.choice(FRACS, size=rng.integers(0, 3), replace=False)),
                               key=Fraction) for k in workloads.CONTEXTS}
    spec["allin"] = {k: bool(rng.random() < 0.7) for k in workloads.CONTEXTS}
    spec["pot"] = int(rng.choice([2, 4, 10, 100]))
    spec["stack"] = int(spec["pot"] * rng.choice([1, 2, 3, 5]))
    spec["raise_cap"] = int(rng.choice([1, 2, 3]))
    spec["open_fold"] = bool(rng.random() < 0.5)
    return spec


@pytest.mark.parametrize("case", range(24))
def test_random_river_configurations(case):
    rng = np.random.default_rng(1000 + case)
    n_ranks, n_suits = [(13, 4), (9, 4), (13, 3), (7, 4), (6, 2), (10, 3), (13, 2), (8, 3)][case % 8]
    spec = random_spec(rng)
    pair = Pair("river", n_games=2, spec=spec, seed=int(rng.integers(1 << 30)), n_ranks=n_ranks, n_suits=n_suits,
                build_sparse=False)
    G = pair.game
    for p in (0, 1):
        o = 1 - p
        blocks = np.zeros((G.n_games, G.n_pub[o] * G.H_pad))
        vals = {}
        for g in range(G.n_games):
            v = pair.tp(g, o).behavioral_to_sequence(random_behavioral(pair.tp(g, o), rng))
            vals[g] = v
            blocks[g] = pair.to_product(g, o, v, row0=1.0)
        dout = torch.full((G.n_games,) + G.vec_shape(p)[1:], np.nan, dtype=torch.float64, device="cuda")
        G.egt_gradient(p, torch.tensor(blocks.reshape((G.n_games,) + G.vec_shape(o)[1:]), device="cuda"), dout)
        torch.cuda.synchronize()
        out = dout.cpu().numpy().reshape(G.n_games, -1)
        for g in range(G.n_games):
            want = pair.sf[g].Ay(vals[g]) if p == 0 else pair.sf[g].ATx(vals[g])
            got = pair.from_product(g, p, out[g])
            got[0] = out[g][:G.H_pad].sum()
            assert_parity(got, want, TOL, "fuzz gradient")
    # one EGT/as iteration from an explicit mu, game 1
    import paper_1810_03063_b200 as P
    sf = pair.sf[1]
    mu = egt.theory_mu(sf) * 2.0 ** -3
    G.egt_init(P.EGT_AS, mu, mu)
    G.egt_step(1)
    sc = G.egt_scalars()
    xs = torch.zeros(G.vec_shape(0), dtype=torch.float64, device="cuda")
    G.get_strategy_device(0, 0, xs)
    prob = egt.Problem(sf)
    x, y = egt.initialize(prob, mu, mu)
    st = egt.EGTState(x, y, mu, mu)
    for _ in range(int(sc[1, 3])):
        egt.egt_iteration(prob, st, "as")
    got = pair.from_product(1, 0, xs.cpu().numpy().reshape(G.n_games, -1)[1])
    assert_parity(got[1:], st.x[1:], TOL, "fuzz egt/as x")


@pytest.mark.parametrize("case", range(8))
def test_random_configurations_cfr_and_fp32(case):
    """The same random configurations: CFR+ averages after 3 iterations (fp64, 1e-9) and the
    fp32 mode's gradients (1e-5, DESIGN.md row 9)."""
    import paper_1810_03063_b200 as P
    from oracle import cfr
    rng = np.random.default_rng(5000 + case)
    n_ranks, n_suits = [(13, 4), (9, 4), (13, 3), (7, 4), (6, 2), (10, 3), (13, 2), (8, 3)][case]
    spec = random_spec(rng)
    seed = int(rng.integers(1 << 30))
    pair = Pair("river", n_games=2, spec=spec, seed=seed, n_ranks=n_ranks, n_suits=n_suits, build_sparse=False)
    G = pair.game
    G.cfr_init(P.CFR_PLUS)
    G.cfr_step(3)
    st = cfr.run(pair.sf[0], "cfr_plus", 3)
    for p, want in ((0, st.xbar), (1, st.ybar)):
        d = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        G.get_strategy_device(p, 1, d)
        got = pair.from_product(0, p, d.cpu().numpy().reshape(G.n_games, -1)[0])
        assert_parity(got[1:], want[1:], TOL, "fuzz cfr+ avg")
    G32 = P.Game(P.RIVER, n_games=2, river=spec, boards=pair.boards, prior1=pair.priors[0], prior2=pair.priors[1],
                 n_ranks=n_ranks, n_suits=n_suits, precision="f32")
    for p in (0, 1):
        o = 1 - p
        v = pair.tp(0, o).behavioral_to_sequence(random_behavioral(pair.tp(0, o), rng))
        blk = np.zeros((2, G.n_pub[o] * G.H_pad))
        blk[0] = pair.to_product(0, o, v, row0=1.0)
        blk[1, :G.H] = 1.0
        dout = torch.zeros((2,) + G.vec_shape(p)[1:], dtype=torch.float32, device="cuda")
        G32.egt_gradient(p, torch.tensor(blk.reshape((2,) + G.vec_shape(o)[1:]), dtype=torch.float32, device="cuda"),
                         dout)
        torch.cuda.synchronize()
        out = dout.double().cpu().numpy().reshape(2, -1)[0]
        want = pair.sf[0].Ay(v) if p == 0 else pair.sf[0].ATx(v)
        got = pair.from_product(0, p, out)
        got[0] = out[:G.H_pad].sum()
        assert_parity(got, want, 1e-5, "fuzz fp32 gradient")
    G32.close()
