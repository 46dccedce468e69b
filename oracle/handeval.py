"""Poker hand evaluator (oracle side), numpy-vectorised, written from the rules.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:686-688: "In a showdown the player with the better hands wins the pot.
The pot is split in case of a tie."  The hand ranking is standard poker's:
straight flush > four of a kind > full house > flush > straight > three of a
kind > two pair > one pair > high card, ties broken by the ranks of the groups
(larger groups first, then higher rank), a straight by its top card, the wheel
A-2-3-4-5 being the lowest straight.  The best 5 of 7 cards counts.

Pins (tests/test_oracle_handeval.py): the textbook frequency of every category
over all C(52,5) five-card hands, and hand-picked orderings.
"""
import itertools

import numpy as np

CATEGORY_NAMES = ["high card", "pair", "two pair", "trips", "straight", "flush",
                  "full house", "quads", "straight flush"]


def eval5(ranks, suits):
    """Strength key of 5-card hands; larger is better, equal means a tie.

    ranks: int array (N, 5), rank values 0..12 (12 = ace); suits: int array (N, 5).
    """
    ranks = np.asarray(ranks, dtype=np.int64)
    suits = np.asarray(suits, dtype=np.int64)
    n = ranks.shape[0]
    rows = np.arange(n)
    counts = np.zeros((n, 13), dtype=np.int64)
    for k in range(5):
        np.add.at(counts, (rows, ranks[:, k]), 1)
    present = counts > 0
    flush = (suits == suits[:, :1]).all(axis=1)

    # straight: highest r with ranks r-4..r all present; the wheel tops at 5 (value 3)
    top = np.full(n, -1, dtype=np.int64)
    for r in range(4, 13):
        top = np.where(present[:, r - 4:r + 1].all(axis=1), r, top)
    wheel = present[:, [12, 0, 1, 2, 3]].all(axis=1)
    top = np.where((top < 0) & wheel, 3, top)
    straight = top >= 0

    # rank groups ordered by (count desc, rank desc)
    order_key = counts * 16 + np.arange(13)[None, :]
    idx = np.argsort(-order_key, axis=1, kind="stable")[:, :5]
    cnt_sorted = np.take_along_axis(counts, idx, axis=1)
    tiebreak = np.where(cnt_sorted > 0, idx, 0)
    c0, c1 = cnt_sorted[:, 0], cnt_sorted[:, 1]

    cat = np.zeros(n, dtype=np.int64)
    cat = np.where(c0 == 2, 1, cat)
    cat = np.where((c0 == 2) & (c1 == 2), 2, cat)
    cat = np.where(c0 == 3, 3, cat)
    cat = np.where(straight, 4, cat)
    cat = np.where(flush, 5, cat)
    cat = np.where((c0 == 3) & (c1 == 2), 6, cat)
    cat = np.where(c0 == 4, 7, cat)
    cat = np.where(straight & flush, 8, cat)

    is_straight_cat = (cat == 4) | (cat == 8)
    tiebreak = np.where(is_straight_cat[:, None],
                        np.concatenate([top[:, None], np.zeros((n, 4), np.int64)], axis=1),
                        tiebreak)
    key = cat * 13 ** 5
    for i in range(5):
        key = key + tiebreak[:, i] * 13 ** (4 - i)
    return key


def category(key):
    return np.asarray(key) // 13 ** 5


def best_of(ranks, suits):
    """Best 5-card key among all 5-subsets of k >= 5 cards. ranks/suits: (N, k)."""
    ranks = np.asarray(ranks)
    suits = np.asarray(suits)
    k = ranks.shape[1]
    best = None
    for sub in itertools.combinations(range(k), 5):
        sub = list(sub)
        key = eval5(ranks[:, sub], suits[:, sub])
        best = key if best is None else np.maximum(best, key)
    return best


def holdem_strengths(deck, board, hands):
    """Showdown key of each 2-card hand with the 5-card board."""
    cards = np.array([list(h) + list(board) for h in hands], dtype=np.int64)
    ranks = 13 - deck.n_ranks + cards // deck.n_suits
    suits = cards % deck.n_suits
    return best_of(ranks, suits)
