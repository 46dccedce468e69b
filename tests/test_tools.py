"""The measurement drivers under tools/ (CPU: they import, and the sweep's bet abstractions
are valid river specs of strictly growing size -- checked with the oracle's own tree builder)."""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_tools_import():
    for m in ("grad_sweep", "convergence", "profile_step", "ncu_summary"):
        if m == "ncu_summary":
            continue  # a script that reads a report at import time
        importlib.import_module(m)


def test_grad_sweep_abstractions_grow():
    from oracle import river
    import grad_sweep
    sizes = []
    for _, spec in grad_sweep.specs():
        rp = river.RiverParams(**{k: spec[k] for k in ("pot", "stack", "fracs", "allin", "raise_cap", "open_fold")})
        tree = river.betting_tree(rp)
        sizes.append((river.PublicSeqs(tree, 0).n_pub, len(river.terminals(tree))))
    assert all(a < b for a, b in zip(sizes, sizes[1:])), sizes
    assert sizes[2] == (152, 203)  # the paper's abstraction: 153 sequences incl. the empty one
