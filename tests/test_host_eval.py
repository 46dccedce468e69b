"""Host-side hand evaluation of the CUDA path's loader (csrc/game.cpp): the direct 7-card
evaluator agrees with the brute-force 5-subset maximum (compiled with g++, CPU only)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_direct_evaluator_matches_subset_maximum(tmp_path):
    exe = tmp_path / "hs_check"
    csrc = os.path.join(ROOT, "paper_1810_03063_b200", "csrc")
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", "-I", os.path.join(ROOT, "include"), "-I", csrc,
                    os.path.join(ROOT, "tests", "cpp", "hand_strength_check.cpp"), os.path.join(csrc, "game.cpp"),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout
    assert "mismatches 0" in out.stdout


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_card_plan_conflict_free_and_exact(tmp_path):
    """The card-domain gradient kernel's host plan (game.cpp build_card_plan) on 48 random
    river boards (one where every hand ties): every shared-memory exchange is bank-conflict
    free per half-warp, delivers each slot its hand's weight and each position its own slots,
    and the run heads / tails / source lanes give the brute-force segment prefixes at the start
    and end of every tie run (index work: exact)."""
    exe = tmp_path / "plan_check"
    csrc = os.path.join(ROOT, "paper_1810_03063_b200", "csrc")
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", "-I", os.path.join(ROOT, "include"), "-I", csrc,
                    os.path.join(ROOT, "tests", "cpp", "card_plan_check.cpp"), os.path.join(csrc, "game.cpp"),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "48"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout
    assert "violations 0" in out.stdout


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_edge_colouring_on_random_multigraphs(tmp_path):
    """The card plan's 16-edge-colouring of bipartite multigraphs (game.cpp colour_edges16: a
    colour free at both ends when one exists, an alternating-path swap otherwise) is proper on
    200 random multigraphs of maximum degree 16, most of them 16-regular with repeated edges --
    the colouring Koenig's theorem guarantees (index work: exact)."""
    exe = tmp_path / "colour_check"
    csrc = os.path.join(ROOT, "paper_1810_03063_b200", "csrc")
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", "-I", os.path.join(ROOT, "include"), "-I", csrc,
                    os.path.join(ROOT, "tests", "cpp", "colour_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "200"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout
    assert "violations 0" in out.stdout
