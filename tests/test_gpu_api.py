"""The public API end to end (paper_1810_03063_b200.solve) and the C ABI's error paths."""
import numpy as np
import pytest

from oracle import br, games, seqform
from paper_1810_03063_b200 import workloads
from tests.paritylib import Pair

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("solver", ["egt_as", "egt_balanced", "cfr_plus", "cfr_rmp"])
def test_solve_kuhn_to_equilibrium(solver):
    """Kuhn poker's value to player 1 is -1/18 (tests/golden/kuhn.json)."""
    import paper_1810_03063_b200 as P
    G = P.Game(P.KUHN, n_games=2)
    sf = seqform.build(games.kuhn())
    res = P.solve(G, solver, eps=2e-3, max_iters=20000, check_every=50)
    assert np.all(res["gap"] <= 2e-3)
    x = res["strategy"][0][0].reshape(-1)
    y = res["strategy"][1][0].reshape(-1)
    pair = Pair("kuhn", n_games=1)
    # host strategy is [n_pub][n_combos]; map to the oracle's sequence space by labels
    Gh = pair.game
    xs = np.zeros((Gh.n_pub[0], Gh.H_pad))
    ys = np.zeros((Gh.n_pub[1], Gh.H_pad))
    xs[:, :3] = x.reshape(Gh.n_pub[0], 3)
    ys[:, :3] = y.reshape(Gh.n_pub[1], 3)
    xv = pair.from_product(0, 0, xs.reshape(-1))
    yv = pair.from_product(0, 1, ys.reshape(-1))
    xv[0] = yv[0] = 1.0
    value = xv @ (sf.A @ yv)          # player 2's expected payoff; the game value is +1/18
    assert abs(value - 1.0 / 18.0) <= 2e-3
    # the reported gap is the oracle's eps_sad of the returned strategies
    assert abs(br.saddle_gap(sf, xv, yv) - res["gap"][0]) <= 1e-9 * max(1.0, res["gap"][0])


def test_solve_river_stops_at_target():
    import paper_1810_03063_b200 as P
    boards = workloads.random_boards(4, 77)
    p1, p2 = workloads.random_priors(boards, 77)
    G = P.Game(P.RIVER, n_games=4, river=workloads.river_spec("simple"), boards=boards, prior1=p1, prior2=p2)
    res = P.solve(G, "egt_as", eps_mbb=200.0, max_iters=3000, check_every=20)
    assert np.all(res["gap"] <= 20.0) and res["iters"] <= 3000
    x, y = res["strategy"]
    assert x.shape == (4, G.n_pub[0], G.n_combos) and y.shape == (4, G.n_pub[1], G.n_combos)
    assert np.all(x >= 0) and np.all(x <= 1 + 1e-12)


def test_error_paths():
    import paper_1810_03063_b200 as P
    G = P.Game(P.KUHN, n_games=1)
    with pytest.raises(P.EGTError):
        G.egt_step(1)                     # before egt_init: EGT_E_STATE
    with pytest.raises(P.EGTError):
        G.cfr_step(1)
    with pytest.raises(P.EGTError):
        G.saddle_gap(0)                   # no solver yet
    d = torch.zeros(G.vec_shape(0), dtype=torch.float64, device="cuda")
    with pytest.raises(P.EGTError):
        G.egt_gradient(2, d, d)           # bad player
    G.egt_init(P.EGT_AS, 1.0, 1.0)
    with pytest.raises(P.EGTError):
        G.shard(0, 1)                     # after init: EGT_E_STATE
    with pytest.raises(P.EGTError):      # invalid board (repeated card)
        P.Game(P.RIVER, n_games=1, river=workloads.river_spec("tiny"), boards=np.array([[1, 1, 2, 3, 4]]))
    with pytest.raises(P.EGTError):      # negative prior
        b = workloads.random_boards(1, 3)
        p1, p2 = workloads.random_priors(b, 3)
        p1[0, np.flatnonzero(p1[0])[0]] = -1.0
        P.Game(P.RIVER, n_games=1, river=workloads.river_spec("tiny"), boards=b, prior1=p1, prior2=p2)
    with pytest.raises(P.EGTError):      # unknown precision
        P.Game(P.KUHN, n_games=1, precision=7)


def test_pool_reuse_and_trim():
    """Game buffers come from the library's device pool: a freed game's memory serves the next
    load, egt_pool_trim hands it back, and a game loaded after the trim computes the same."""
    import torch
    import paper_1810_03063_b200 as P
    boards = workloads.random_boards(4, 77)
    p1, p2 = workloads.random_priors(boards, 77)
    spec = workloads.river_spec("simple")
    gaps = []
    for trim in (False, True, False):
        G = P.Game(P.RIVER, n_games=4, river=spec, boards=boards, prior1=p1, prior2=p2)
        G.egt_init(P.EGT_AS)
        G.egt_step(5)
        gaps.append(G.saddle_gap(0))
        G.close()
        if trim:
            free0 = torch.cuda.mem_get_info()[0]
            P.pool_trim()
            assert torch.cuda.mem_get_info()[0] >= free0
    assert np.array_equal(gaps[0], gaps[1]) and np.array_equal(gaps[1], gaps[2])


def test_batch_independence():
    """A game's EGT/as trajectory does not depend on the batch around it (different chunking,
    launch shapes, masks): games 0 and n-1 of a 300-game batch equal the same games solved
    alone, bit for bit."""
    import paper_1810_03063_b200 as P
    n = 300
    spec = workloads.river_spec("libratus")
    boards = workloads.random_boards(n, 99)
    p1, p2 = workloads.random_priors(boards, 99)
    G = P.Game(P.RIVER, n_games=n, river=spec, boards=boards, prior1=p1, prior2=p2)
    G.egt_init(P.EGT_AS)
    G.egt_step(3)
    gap = G.saddle_gap(0)
    sc = G.egt_scalars()
    G.close()
    for i in (0, n - 1):
        G1 = P.Game(P.RIVER, n_games=1, river=spec, boards=boards[i:i + 1], prior1=p1[i:i + 1], prior2=p2[i:i + 1])
        G1.egt_init(P.EGT_AS)
        G1.egt_step(3)
        assert G1.saddle_gap(0)[0] == gap[i]
        assert np.array_equal(G1.egt_scalars()[0, :7], sc[i, :7])
        G1.close()


def test_device_stopping_target():
    """egt_set_target: a game whose eps_sad reached its target stops on the device (its
    iterate, counters and gap freeze); the others follow exactly the trajectory of a run
    without targets; clearing the targets resumes the stopped games."""
    import paper_1810_03063_b200 as P
    n, k = 12, 60
    spec = workloads.river_spec("simple")
    boards = workloads.random_boards(n, 31)
    p1, p2 = workloads.random_priors(boards, 31)

    def run(target):
        G = P.Game(P.RIVER, n_games=n, river=spec, boards=boards, prior1=p1, prior2=p2)
        G.egt_init(P.EGT_AS)
        if target is not None:
            G.egt_set_target(target)
        G.egt_step(k)
        return G, G.saddle_gap(0), G.egt_scalars()

    G0, gap0, sc0 = run(None)
    G0.close()
    eps = float(np.median(gap0)) * 1.5  # some games get there within k iterations, some not
    G1, gap1, sc1 = run(eps)
    attempts0, attempts1 = sc0[:, 4], sc1[:, 4]
    stopped = attempts1 < k
    assert stopped.any() and not stopped.all()
    assert np.all(gap1[stopped] <= eps)
    assert np.array_equal(gap1[~stopped], gap0[~stopped])
    assert np.array_equal(sc1[~stopped, :7], sc0[~stopped, :7])
    # a stopped game froze at the first iteration its gap was <= eps: iterating further never
    # happened, so one more block of steps changes nothing for it
    G1.egt_step(5)
    assert np.array_equal(G1.egt_scalars()[stopped, :7], sc1[stopped, :7])
    G1.egt_set_target(None)
    G1.egt_step(5)
    assert np.all(G1.egt_scalars()[stopped, 4] == sc1[stopped, 4] + 5)
    G1.close()


def test_cfr_stopping_target():
    """CFR with egt_set_target: a game stops at the first saddle_gap evaluation of its average
    that finds eps_sad <= its target; the others run exactly as without targets."""
    import paper_1810_03063_b200 as P
    n, checks, every = 10, 6, 10
    spec = workloads.river_spec("simple")
    boards = workloads.random_boards(n, 41)
    p1, p2 = workloads.random_priors(boards, 41)

    def run(target):
        G = P.Game(P.RIVER, n_games=n, river=spec, boards=boards, prior1=p1, prior2=p2)
        G.cfr_init(P.CFR_PLUS)
        if target is not None:
            G.egt_set_target(target)
        hist = []
        for _ in range(checks):
            G.cfr_step(every)
            hist.append(G.saddle_gap(1))
        t = G.egt_scalars()[:, 3]
        G.close()
        return np.array(hist), t

    h0, t0 = run(None)
    eps = float(np.median(h0[-1]))  # about half the games get there within the run
    h1, t1 = run(eps)
    first = [next((c for c in range(checks) if h0[c, g] <= eps), None) for g in range(n)]
    assert any(f is not None for f in first) and any(f is None for f in first)
    for g, f in enumerate(first):
        if f is None:
            assert np.array_equal(h1[:, g], h0[:, g]) and t1[g] == t0[g]
        else:
            assert np.array_equal(h1[:f + 1, g], h0[:f + 1, g])   # identical until it stopped
            assert np.all(h1[f:, g] == h0[f, g])                   # then frozen
            assert t1[g] == 1 + every * (f + 1)
