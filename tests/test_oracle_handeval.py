"""Pins for oracle/handeval.py (no GPU)."""
import itertools
import json
import os

import numpy as np

from oracle.handeval import CATEGORY_NAMES, category, eval5, best_of

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_five_card_category_counts():
    """Textbook frequencies over all C(52,5) hands (tests/golden/handeval_5card_counts.json)."""
    want = json.load(open(os.path.join(GOLD, "handeval_5card_counts.json")))["counts"]
    c = np.array(list(itertools.combinations(range(52), 5)), dtype=np.int64)
    got = np.bincount(category(eval5(c // 4, c % 4)), minlength=9)
    assert {CATEGORY_NAMES[i]: int(got[i]) for i in range(9)} == want


def _key(cards):
    """cards like 'As Kd ...' -> key."""
    R = "23456789TJQKA"
    S = "cdhs"
    r = [[R.index(x[0]) for x in cards.split()]]
    s = [[S.index(x[1]) for x in cards.split()]]
    return int(best_of(np.array(r), np.array(s))[0])


def test_orderings():
    assert _key("Ah Kh Qh Jh Th") > _key("Kh Qh Jh Th 9h")          # straight flushes by top
    assert _key("5c 4d 3h 2s Ac") < _key("6c 5d 4h 3s 2c")          # the wheel is the lowest straight
    assert _key("As Ad Kc 2h 3h") > _key("As Ad Qc Jh Th")          # pair: kicker
    assert _key("3s 3d 3c 2h 2d") < _key("4s 4d 4c 2h 2d")          # full houses by trips
    assert _key("Ks Kd 2c 2h 7d") > _key("Qs Qd Jc Jh Ad")          # two pair: top pair first
    assert _key("2h 4h 6h 8h Th") > _key("Ac Kd Qh Js Tc")          # flush beats straight
    assert _key("As Ks Qd Jc 9h") == _key("Ah Kh Qc Jd 9s")         # suits never break ties
    # best 5 of 7: board plays (tie)
    assert _key("2c 3d Ah Kh Qh Jh Th") == _key("4c 5d Ah Kh Qh Jh Th")
