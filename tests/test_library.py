"""The C ABI library builds for sm_100a, loads, and exports every symbol the header declares (no GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1810_03063_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "egt_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\**\s*(\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib_path():
    return B.build()


def test_header_declares_the_boundary():
    names = header_functions()
    for want in ("egt_load_game", "egt_init", "egt_step", "cfr_init", "cfr_step", "saddle_gap",
                 "get_avg_strategy", "egt_gradient", "egt_smoothed_br", "egt_prox", "egt_best_response"):
        assert want in names


def test_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    assert set(header_functions()) <= exported


def test_built_for_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_fails_loudly_without_device(lib_path):
    """No CPU fallback: without a CUDA device, loading a game raises."""
    import paper_1810_03063_b200 as P
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(P.EGTError):
        P.Game(P.KUHN)


def test_every_declaration_cites_its_passage():
    """SURVEY-less §8(b): each exported call's comment cites the PAPER.md passage that defines
    the operation (or, for plumbing, the passage whose data it handles)."""
    src = open(os.path.join(ROOT, "include", "egt_b200.h")).read()
    decls = [(m.start(), m.group(1)) for m in re.finditer(r"^(?:int|void|const char\*)\s+(\w+)\(", src, re.M)]
    assert len(decls) == len(header_functions())
    prev = 0
    missing = []
    for pos, name in decls:
        chunk = src[prev:pos]
        comment = chunk[chunk.rfind("/*"):] if "/*" in chunk else ""
        if "PAPER.md:" not in comment:
            missing.append(name)
        prev = pos
    assert not missing, missing
