"""Row 8: one game sharded over ranks by terminal rows, NCCL all-reduce per gradient.

On one GPU the ranks cannot run concurrently (B200_PROFILING.md), so the sharded
arithmetic is checked by emulation -- every rank's slice computed on the same device
(egt_gradient_rows) must sum, bit for bit, to the unsharded gradient -- and the NCCL path
itself runs with a 1-rank communicator inside the solver's CUDA graph."""
import numpy as np
import pytest

from paper_1810_03063_b200 import workloads
from tests.paritylib import Pair

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _random_vec(G, p, seed):
    rng = np.random.default_rng(seed)
    v = rng.random((G.n_games, G.n_pub[p], G.H_pad))
    v[:, :, G.H:] = 0.0
    v[:, 0, :G.H] = 1.0
    return torch.tensor(v, dtype=torch.float64, device="cuda")


@pytest.mark.parametrize("kind,world", [("river", 2), ("river", 3), ("river", 8), ("leduc", 2), ("kuhn", 3),
                                        ("libratus", 8)])
def test_slices_sum_to_full_gradient(kind, world):
    if kind == "libratus":
        pair = Pair("river", n_games=4, spec=workloads.river_spec("libratus"), seed=5, sample=[])
    elif kind == "river":
        pair = Pair("river", n_games=3, seed=2, sample=[])
    else:
        pair = Pair(kind, n_games=2)
    G = pair.game
    for p in (0, 1):
        din = _random_vec(G, 1 - p, 10 + p)
        full = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        G.egt_gradient(p, din, full)
        acc = torch.zeros_like(full)
        touched = torch.zeros_like(full, dtype=torch.int32)
        for r in range(world):
            part = torch.full_like(full, np.nan)
            G.gradient_rows(p, r, world, din, part)
            assert torch.isfinite(part).all()
            touched += (part != 0).int()
            acc += part
        assert torch.equal(acc, full)           # disjoint rows: the sum is exact
        assert int(touched.max()) <= 1          # no row computed by two ranks


def test_nccl_unique_id():
    import paper_1810_03063_b200 as P
    uid = P.binding.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == P.binding.NCCL_ID_BYTES


@pytest.mark.parametrize("solver", ["egt_as", "cfr_plus"])
def test_one_rank_nccl_solver_is_identical(solver):
    """The sharded solver with a real (1-rank) NCCL communicator inside the CUDA graph
    reproduces the unsharded solver exactly."""
    import paper_1810_03063_b200 as P
    spec = workloads.river_spec("simple")
    boards = workloads.random_boards(4, 31)
    p1, p2 = workloads.random_priors(boards, 31)
    games = []
    for sharded in (False, True):
        G = P.Game(P.RIVER, n_games=4, river=spec, boards=boards, prior1=p1, prior2=p2)
        if sharded:
            G.shard(0, 1, uid=P.binding.nccl_unique_id())
        if solver == "egt_as":
            G.egt_init(P.EGT_AS, 50.0, 50.0)
            G.egt_step(6)
        else:
            G.cfr_init(P.CFR_PLUS)
            G.cfr_step(6)
        games.append(G)
    for p in (0, 1):
        a = torch.zeros(games[0].vec_shape(p), dtype=torch.float64, device="cuda")
        b = torch.zeros_like(a)
        games[0].get_strategy_device(p, 1, a)
        games[1].get_strategy_device(p, 1, b)
        assert torch.equal(a, b)
    assert np.array_equal(games[0].saddle_gap(1), games[1].saddle_gap(1))
    kt = None
    games[1].timing(True)
    if solver == "egt_as":
        games[1].egt_step(1)
    else:
        games[1].cfr_step(1)
    kt = games[1].timing_get()
    games[1].timing(False)
    assert kt["comm"][1] >= 2                    # the all-reduces ran


def test_kernel_timing_accounting():
    """egt_timing: eager launches bracketed by events; per kind the launches, the game-launches
    that did work and the algorithmic bytes add up for one EGT/as iteration."""
    import paper_1810_03063_b200 as P
    spec = workloads.river_spec("simple")
    boards = workloads.random_boards(3, 41)
    p1, p2 = workloads.random_priors(boards, 41)
    G = P.Game(P.RIVER, n_games=3, river=spec, boards=boards, prior1=p1, prior2=p2)
    G.egt_init(P.EGT_AS, 30.0, 30.0)
    G.timing(True)
    G.egt_step(1)
    kt = G.timing_get()
    G.timing(False)
    # per game: 4 gradients (2 on the focused player's launches, 2 in the excessive-gap check)
    grads = kt["grad_Ay"][2] + kt["grad_ATx"][2]
    assert grads == 4 * 3
    assert kt["grad_Ay"][1] + kt["grad_ATx"][1] == 6          # 4 masked + 2 full launches
    # bytes: 8 H (R_r + R_w + 2) per game-gradient, + 8 H R_r where the input x_hat is formed from
    # two vectors' rows (the first gradient of each focus chain, Alg. 2 line 1 fused)
    per_game = [8 * G.H * (G.grad_rows_read[p] + G.grad_rows_written[p] + 2) for p in (0, 1)]
    extra = [8 * G.H * G.grad_rows_read[p] for p in (0, 1)]
    for p, k in ((0, "grad_Ay"), (1, "grad_ATx")):
        assert per_game[p] * kt[k][2] - 1e-6 <= kt[k][3] <= (per_game[p] + extra[p]) * kt[k][2] + 1e-6
    assert kt["tree"][1] == 6 and kt["tree"][0] > 0 and kt["tree"][3] > 0  # 4 masked + 2 EGC (SBR + fused BR)
    assert kt["scalar"][1] == 2 and kt["comm"][1] == 0
    G.egt_step(2)  # back on the CUDA graph
    assert np.isfinite(G.saddle_gap(0)).all()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_fused_allgather_stores_emulated(world):
    """The fused kernel stores each shard's rows into every shard's buffer: after all emulated
    ranks ran (one device, no waiting between them), every buffer equals the full gradient."""
    pair = Pair("river", n_games=3, spec=workloads.river_spec("libratus"), seed=12, sample=[])
    G = pair.game
    for p in (0, 1):
        din = _random_vec(G, 1 - p, 50 + p)
        full = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
        G.egt_gradient(p, din, full)
        bufs = [torch.zeros_like(full) for _ in range(world)]
        for r in range(world):
            G.gradient_rows_to(p, r, world, din, bufs)
        for b in bufs:
            assert torch.equal(b, full)


def test_fused_allgather_solver_one_rank():
    """egt_shard + egt_shard_peers (IPC handles of this rank) runs the solver with the fused
    gradient stores and the one-element NCCL barrier inside the graph: identical results."""
    import paper_1810_03063_b200 as P
    spec = workloads.river_spec("simple")
    boards = workloads.random_boards(3, 33)
    p1, p2 = workloads.random_priors(boards, 33)
    res = []
    for fused in (False, True):
        G = P.Game(P.RIVER, n_games=3, river=spec, boards=boards, prior1=p1, prior2=p2)
        if fused:
            G.shard(0, 1, uid=P.binding.nccl_unique_id())
            G.shard_peers([G.ipc_handles()])
        G.egt_init(P.EGT_AS, 40.0, 40.0)
        G.egt_step(5)
        x = torch.zeros(G.vec_shape(0), dtype=torch.float64, device="cuda")
        G.get_strategy_device(0, 0, x)
        res.append((x.cpu().numpy(), G.saddle_gap(0)))
        if fused:
            G.timing(True)
            G.egt_step(1)
            kt = G.timing_get()
            G.timing(False)
            assert kt["comm"][1] >= 4 and kt["comm"][3] == 0      # barriers, no all-reduced bytes
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


# ------------------------------------------------------------------ emulated ranks, whole solver
@pytest.mark.parametrize("solver", ["egt_as", "cfr_plus"])
@pytest.mark.parametrize("world,fused", [(2, False), (3, False), (8, False), (2, True), (3, True)])
def test_emulated_ranks_solver(world, fused, solver):
    """The sharded SOLVER path on `world` emulated ranks (egt_shard_emulate): every gradient
    runs each rank's slice kernel into that rank's own (reused) buffer, then the collective
    (a local sum for the NCCL all-reduce, or the fused kernels' stores into every rank's
    buffer).  Five EGT/as attempts (30 consecutive gradients) or five CFR+ iterations must equal the unsharded solver bit for bit
    and the oracle at 1e-9.  Before the non-owned rows were zeroed, the all-reduce variant
    summed stale rows of the previous gradient from the second gradient on."""
    import paper_1810_03063_b200 as P
    from oracle import br, cfr, egt
    from tests.paritylib import assert_parity, assert_scalar
    spec = workloads.river_spec("tiny", pot=2, stack=6, raise_cap=2)
    pair = Pair("river", n_games=2, spec=spec, seed=21)
    runs = []
    for emulate in (False, True):
        G = P.Game(P.RIVER, n_games=2, river=spec, boards=pair.boards, prior1=pair.priors[0],
                   prior2=pair.priors[1])
        if emulate:
            G.shard_emulate(world, fused)
        if solver == "egt_as":
            mu = egt.theory_mu(pair.sf[0]) / 8.0
            G.egt_init(P.EGT_AS, mu, mu)
            G.egt_step(5)
            which = 0
        else:
            G.cfr_init(P.CFR_PLUS)
            G.cfr_step(5)
            which = 1
        vecs = []
        for p in (0, 1):
            d = torch.zeros(G.vec_shape(p), dtype=torch.float64, device="cuda")
            G.get_strategy_device(p, which, d)
            vecs.append(d.cpu().numpy())
        runs.append((vecs, G.saddle_gap(which), G.egt_scalars()))
    (v0, g0, s0), (v1, g1, s1) = runs
    assert all(np.array_equal(a, b) for a, b in zip(v0, v1))
    assert np.array_equal(g0, g1)
    cols = slice(0, 7) if solver == "egt_as" else slice(3, 4)  # CFR keeps only t among the scalars
    assert np.array_equal(s0[:, cols], s1[:, cols])
    sf = pair.sf[0]
    if solver == "egt_as":
        prob = egt.Problem(sf)
        x, y = egt.initialize(prob, mu, mu)
        st = egt.EGTState(x, y, mu, mu)
        for _ in range(int(s1[0, 3])):
            egt.egt_iteration(prob, st, "as")
        assert int(s1[0, 5]) == st.backtracks
        want = (st.x, st.y)
    else:
        st = cfr.run(sf, "cfr_plus", 5)
        want = (st.xbar, st.ybar)
    for p in (0, 1):
        assert_parity(pair.from_product(0, p, v1[p].reshape(2, -1)[0])[1:], want[p][1:], 1e-9,
                      "emulated-rank solver")
    assert_scalar(g1[0], br.saddle_gap(sf, *want), 1e-9, "emulated-rank solver eps_sad")
