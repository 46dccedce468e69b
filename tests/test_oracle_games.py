"""Pins for oracle/treeplex.py, oracle/games.py, oracle/seqform.py, oracle/river.py (no GPU)."""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import games, seqform, river
from oracle.cards import Deck
from oracle.treeplex import Treeplex
from paper_1810_03063_b200 import workloads

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def fig1():
    g = json.load(open(os.path.join(GOLD, "fig1_treeplex.json")))
    simplexes, nxt = [], 1
    for dim, par in g["simplexes_1based"]:
        simplexes.append((nxt, dim, 0 if par == "root" else par))
        nxt += dim
    return Treeplex(nxt, simplexes), g["expected"]


def vertices(tp):
    """All pure strategies of a small treeplex, in sequence form."""
    choices = [range(tp.size[j]) for j in range(tp.n_simplex)]
    out = []
    for pick in itertools.product(*choices):
        b = np.zeros(tp.n_seq)
        b[0] = 1
        for j, i in enumerate(pick):
            b[tp.start[j] + i] = 1
        out.append(tp.behavioral_to_sequence(b))
    return out


def random_treeplex(rng, n_simplex):
    simplexes, nxt = [], 1
    for _ in range(n_simplex):
        dim = int(rng.integers(1, 4))
        par = 0 if nxt == 1 or rng.random() < 0.3 else int(rng.integers(1, nxt))
        simplexes.append((nxt, dim, par))
        nxt += dim
    return Treeplex(nxt, simplexes)


# ------------------------------------------------------------------ treeplex
def test_fig1_values():
    tp, want = fig1()
    for j, v in want["b"].items():
        assert tp.b[int(j) - 1] == v
    for j, v in want["d"].items():
        assert tp.d[int(j) - 1] == v
    assert tp.start[0] == 1 and tp.size[0] == 2 and tp.start[1] == 3 and tp.size[1] == 3  # I_1, I_2


def test_beta_recurrence_small():
    # root Delta_2 whose action 1 leads to one leaf Delta_2: beta_leaf = 2, beta_root = 2 + 2*2
    tp = Treeplex(5, [(1, 2, 0), (3, 2, 1)])
    assert tp.beta[1] == 2 and tp.beta[0] == 6


@pytest.mark.parametrize("seed", range(6))
def test_M_and_Omega_by_vertex_enumeration(seed):
    """M = max ||q||_1 and Omega = max d - min d (min 0 at the centre) over Q; both
    attained at vertices for M (linear) and for d (convex)."""
    from oracle.dgf import dgf_value
    tp = random_treeplex(np.random.default_rng(seed), 6)
    V = vertices(tp)
    assert math.isclose(tp.M, max(v[1:].sum() for v in V), rel_tol=1e-12)
    assert math.isclose(tp.Omega, max(dgf_value(tp, v) for v in V), rel_tol=1e-12)
    assert abs(dgf_value(tp, tp.uniform())) < 1e-12


def test_round_trip_and_uniform():
    tp, _ = fig1()
    rng = np.random.default_rng(0)
    b = tp.uniform_behavioral()
    for j in range(tp.n_simplex):
        s, n = tp.start[j], tp.size[j]
        w = rng.random(n) + 0.1
        b[s:s + n] = w / w.sum()
    q = tp.behavioral_to_sequence(b)
    assert tp.check_feasible(q)
    assert np.allclose(tp.behavioral_to_sequence(tp.sequence_to_behavioral(q)), q, atol=1e-12)
    u = tp.uniform()
    assert np.allclose(u[1:3], 0.5) and np.allclose(u[3:6], 1 / 3)
    assert np.allclose(u[6:8], 0.25)  # Delta_3 under q_1: 0.5 * 1/2


def test_invalid_treeplexes():
    with pytest.raises(ValueError):
        Treeplex(3, [(1, 2, 2)])          # parent inside itself (cycle)
    with pytest.raises(ValueError):
        Treeplex(4, [(1, 2, 0)])          # index 3 uncovered


# ------------------------------------------------------------------ sequence form
def test_matching_pennies():
    sf = seqform.build(games.matrix_game([[1, -1], [-1, 1]]))
    A = sf.A.toarray()
    assert np.allclose(A[1:, 1:], -np.array([[1, -1], [-1, 1]]))
    assert sf.max_abs_A() == 1.0


def test_kuhn_shape():
    g = json.load(open(os.path.join(GOLD, "kuhn.json")))
    sf = seqform.build(games.kuhn())
    assert sf.X.n_simplex == sf.Y.n_simplex == g["infosets_per_player"]
    assert sf.X.n_seq == g["sequences_per_player_incl_empty"]


def _random_behavioral(tp, rng):
    b = tp.uniform_behavioral()
    for j in range(tp.n_simplex):
        s, n = tp.start[j], tp.size[j]
        w = rng.random(n) ** 2
        b[s:s + n] = w / w.sum()
    return b


def _tree_walk_check(root, sf, rng, trials):
    for _ in range(trials):
        bx = _random_behavioral(sf.X, rng)
        by = _random_behavioral(sf.Y, rng)
        B = [bx, by]
        # behavioural probabilities per information set (hand, history before the action),
        # recovered from the label "hand|history/action" of the simplex's first sequence
        cache = [{}, {}]
        for p, tp, labels in ((0, sf.X, sf.labels_x), (1, sf.Y, sf.labels_y)):
            for j in range(tp.n_simplex):
                s, n = tp.start[j], tp.size[j]
                hand, hist = labels[s].split("|", 1)
                before = hist[:hist.rfind("/")] if "/" in hist else ""
                cache[p][(hand, before)] = B[p][s:s + n]

        def strat(player, hand, hist):
            return cache[player][(hand, hist)]
        x = sf.X.behavioral_to_sequence(bx)
        y = sf.Y.behavioral_to_sequence(by)
        want = -games.expected_payoff1(root, strat)
        got = x @ (sf.A @ y)
        assert abs(got - want) <= 1e-10 * max(1.0, sf.max_abs_A())


@pytest.mark.parametrize("name", ["kuhn", "leduc"])
def test_xAy_equals_tree_walk(name):
    root = getattr(games, name)()
    sf = seqform.build(root)
    _tree_walk_check(root, sf, np.random.default_rng(1), 30 if name == "leduc" else 200)


# ------------------------------------------------------------------ river rules
def test_river_tiny_tree_matches_hand_enumeration():
    g = json.load(open(os.path.join(GOLD, "river_tiny_tree.json")))
    rp = river.RiverParams(pot=2, stack=4, fracs={k: ["1"] for k in river.CONTEXTS},
                           allin={k: True for k in river.CONTEXTS}, raise_cap=2, open_fold=False)
    tree = river.betting_tree(rp)
    nodes = [{}, {}]
    terms = {}

    def rec(n):
        if n.kind == "terminal":
            if n.fold_by is not None:
                terms[n.history] = ["fold_p%d" % (n.fold_by + 1), n.payoff_fold_to_p1]
            else:
                terms[n.history] = ["showdown", n.showdown_amount]
            return
        nodes[n.player][n.history] = [t for t, _ in n.children]
        for _, c in n.children:
            rec(c)
    rec(tree)
    assert terms == g["terminals"]
    assert nodes[0] == g["p1_nodes"] and nodes[1] == g["p2_nodes"]


def test_libratus_raise_chains_match_hand_enumeration():
    """Deep raise chains of the Libratus abstraction: every context incl. the "subsequent
    raises" lists of both players at the nodes of two chains, with the bet
    totals and payoffs derived by hand (tests/golden/river_libratus_raise_chains.json)."""
    g = json.load(open(os.path.join(GOLD, "river_libratus_raise_chains.json")))
    spec = workloads.river_spec("libratus")
    rp = river.RiverParams(**{k: spec[k] for k in ("pot", "stack", "fracs", "allin", "raise_cap", "open_fold")})
    tree = river.betting_tree(rp)
    by_hist = {}

    def rec(n):
        by_hist[n.history] = n
        for _, c in n.children:
            rec(c)
    rec(tree)
    seen = set()
    for chain in g["chains"]:
        for nd in chain["nodes"]:
            n = by_hist[nd["history"]]
            assert n.kind == "decision" and n.player == nd["player"] - 1
            assert [t for t, _ in n.children] == nd["children"], nd["history"]
            seen.add(river.context(n.player, nd["history"].count("b")))
            assert river.context(n.player, nd["history"].count("b")) == nd["context"]
        for tm in chain["terminals"]:
            n = by_hist[tm["history"]]
            assert n.kind == "terminal"
            if "fold_by" in tm:
                assert n.fold_by == tm["fold_by"] - 1 and n.payoff_fold_to_p1 == tm["payoff_to_p1"]
            else:
                assert n.showdown_amount == tm["showdown_amount"]
    assert seen == set(river.CONTEXTS)


def test_libratus_abstraction_size():
    """Endgame-2-shaped tree: same order as the paper's 140k/144k dims and 176M
    leaves (the paper prunes zero-probability hands)."""
    spec = workloads.river_spec("libratus")
    rp = river.RiverParams(**{k: spec[k] for k in ("pot", "stack", "fracs", "allin", "raise_cap", "open_fold")})
    tree = river.betting_tree(rp)
    p = [river.PublicSeqs(tree, 0), river.PublicSeqs(tree, 1)]
    nt = len(river.terminals(tree))
    dims = [1081 * q.n_pub for q in p]
    assert 120e3 < dims[0] < 200e3 and 120e3 < dims[1] < 200e3
    assert 1.5e8 < nt * 1081 * 990 < 3e8


def _small_river(seed=0, kind="tiny", n_ranks=5):
    deck = Deck(n_ranks, 4)
    board = workloads.random_boards(1, seed, n_ranks, 4)[0]
    p1, p2 = workloads.random_priors([board], seed, n_ranks, 4)
    spec = workloads.river_spec(kind, pot=2, stack=6, raise_cap=2)
    rp = river.RiverParams(**{k: spec[k] for k in ("pot", "stack", "fracs", "allin", "raise_cap", "open_fold")})
    d1 = workloads.prior_dict(p1[0], deck.n_cards)
    d2 = workloads.prior_dict(p2[0], deck.n_cards)
    return rp, deck, board, d1, d2


def test_river_vectorised_equals_literal():
    """The hand-vectorised river sequence form equals the literal tree's A
    entry by entry (aligned by sequence labels), on a 20-card deck."""
    rp, deck, board, d1, d2 = _small_river()
    lit = seqform.build(games.river_literal(rp, deck, board, d1, d2))
    vec = river.RiverSeqForm(rp, deck, board, d1, d2)

    def entries(sf):
        A = sf.A.tocoo()
        return {(sf.labels_x[i], sf.labels_y[j]): v for i, j, v in zip(A.row, A.col, A.data) if v != 0}
    a, b = entries(lit), entries(vec)
    assert a.keys() == b.keys()
    assert max(abs(a[k] - b[k]) for k in a) < 1e-14
    # treeplexes agree on the set of sequences that any leaf reaches
    rng = np.random.default_rng(3)
    y = vec.Y.behavioral_to_sequence(_random_behavioral(vec.Y, rng))
    x = vec.X.behavioral_to_sequence(_random_behavioral(vec.X, rng))
    assert np.allclose(vec.Ay(y), vec.A @ y, rtol=0, atol=1e-13)
    assert np.allclose(vec.ATx(x), vec.A.T @ x, rtol=0, atol=1e-13)
    assert math.isclose(vec.max_abs_A(), np.abs(vec.A.data).max(), rel_tol=1e-14)


def test_river_literal_tree_walk():
    rp, deck, board, d1, d2 = _small_river(seed=4, n_ranks=4)
    root = games.river_literal(rp, deck, board, d1, d2)
    _tree_walk_check(root, seqform.build(root), np.random.default_rng(2), 10)
