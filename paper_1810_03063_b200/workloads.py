"""Seeded synthetic inputs shared by the CUDA path, the oracle tests and bench.py.

This module holds NONE of the method's arithmetic: it only produces the game
parameters (pot, stack, bet-size fractions as exact rational strings) and the
random boards / hand priors of the synthetic workloads.  Both the oracle
(``oracle/``) and the CUDA path (``paper_1810_03063_b200``) consume its plain
outputs; it imports neither.

Recipe:
* Bet abstractions follow PAPER.md:673-685.  ``libratus`` is the paper's full
  fine-grained abstraction; ``simple`` is BASELINE.json configs[2]'s
  {0.5, 1, all-in}; ``tiny`` is a one-size abstraction for brute-force tests.
* Pot/stack: Endgame 2 of PAPER.md:692 has pot 2100; stacks are 200 big blinds
  of 100 chips, so 20000 - 1050 = 18950 behind.
* Boards: 5 distinct cards drawn uniformly (numpy PCG64, seeded).
* Priors ("the conditional distribution over hands"): per
  hole-card combo, weight exp(sigma * N(0,1)) with sigma = 1, and a fraction
  ``zero_frac`` (default 0.15) of combos set to 0 (hands that left the range
  earlier in the hand); combos that touch the board get 0.  Canonical combo
  order: (c1, c2), c1 < c2, lexicographic; card id = rank_pos * n_suits + suit.
"""
import itertools

import numpy as np

CONTEXTS = ("P1_OPEN", "P1_VS_BET", "P1_VS_RAISE", "P1_SUBSEQ",
            "P2_VS_CHECK", "P2_VS_BET", "P2_SUBSEQ")

# PAPER.md:675-685, as (context -> pot multipliers), all contexts allow all-in
LIBRATUS_FRACS = {
    "P1_OPEN": ["1/4", "1/2", "1", "2", "4", "8"],
    "P1_VS_BET": ["2/5", "7/10", "11/10", "2"],
    "P1_VS_RAISE": ["2/5", "7/10", "2"],
    "P1_SUBSEQ": ["7/10"],
    "P2_VS_CHECK": ["1/2", "3/4", "1"],
    "P2_VS_BET": ["7/10", "11/10"],
    "P2_SUBSEQ": ["7/10"],
}


def river_spec(kind="libratus", pot=2100, stack=18950, raise_cap=1000, open_fold=True,
               big_blind=100):
    """Parameters of a river endgame."""
    if kind == "libratus":
        fracs = {k: list(v) for k, v in LIBRATUS_FRACS.items()}
    elif kind == "simple":                      # BASELINE.json configs[2]: {0.5, 1, all-in}
        fracs = {k: ["1/2", "1"] for k in CONTEXTS}
    elif kind == "tiny":
        fracs = {k: ["1"] for k in CONTEXTS}
    else:
        raise ValueError(kind)
    return {
        "pot": int(pot), "stack": int(stack), "fracs": fracs,
        "allin": {k: True for k in CONTEXTS}, "raise_cap": int(raise_cap),
        "open_fold": bool(open_fold), "big_blind": big_blind,
    }


def combos(n_cards):
    return list(itertools.combinations(range(n_cards), 2))


def random_boards(n_games, seed, n_ranks=13, n_suits=4, n_board=5):
    rng = np.random.Generator(np.random.PCG64(seed))
    n_cards = n_ranks * n_suits
    return np.stack([np.sort(rng.choice(n_cards, size=n_board, replace=False))
                     for _ in range(n_games)]).astype(np.int32)


def random_priors(boards, seed, n_ranks=13, n_suits=4, sigma=1.0, zero_frac=0.15):
    """(prior1, prior2), each float64 [n_games, n_combos] in canonical combo order."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    n_cards = n_ranks * n_suits
    cs = np.array(combos(n_cards))
    out = []
    for _player in range(2):
        P = np.exp(sigma * rng.standard_normal((len(boards), len(cs))))
        P *= rng.random((len(boards), len(cs))) >= zero_frac
        for g, b in enumerate(boards):
            blocked = np.isin(cs[:, 0], b) | np.isin(cs[:, 1], b)
            P[g, blocked] = 0.0
        out.append(P)
    return out[0], out[1]


def prior_dict(prior_row, n_cards):
    """Canonical-order prior row -> {(c1, c2): weight} (oracle input form)."""
    return {c: float(w) for c, w in zip(combos(n_cards), prior_row)}
