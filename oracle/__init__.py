"""CPU oracle for arXiv:1810.03063 (EGT with the dilated entropy DGF, and the
CFR(RM) / CFR(RM+) / CFR+ baselines).

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import this package:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs call it.  It shares no code, tables or constants
with ``paper_1810_03063_b200`` (the CUDA path); the two meet only through the
seeded input generators in ``paper_1810_03063_b200/workloads.py`` (which hold
none of the method's arithmetic) and through the canonical labels both sides
emit for sequences (used by the tests to align the two index spaces).

Everything here is plain fp64 numpy / scipy, written to be checked by eye
against PAPER.md (cited as ``PAPER.md:<line>`` with the section/algorithm).

Modules
-------
cards, handeval   deck / hole-card combos and a 5-of-7 poker hand evaluator
games             literal extensive-form game trees (Kuhn, Leduc, river, matrix games)
river             river-endgame betting rules and a
                  hand-vectorised sequence-form builder for full-deck rivers
seqform           treeplexes + sparse sequence-form payoff matrix A from an EFG
treeplex          the treeplex structure
dgf               dilated entropy DGF, smoothed best response, prox
br                best responses and the saddle-point residual
egt               EGT / EGT (mu-balanced) / EGT/as
cfr               Gen-CFR with RM / RM+ and the CFR variants
lp                sequence-form LP (game value pin; not part of the paper's method)

Parity pins are listed in DESIGN.md ("Oracle pins"); every function here has
at least one pin in tests/test_oracle_*.py.
"""
