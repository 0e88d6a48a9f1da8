"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/dma.h declares, and its host-side plan helpers match the oracle."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import mx_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dma.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(dma_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_header_symbols():
    from paper_2604_03950_b200 import _lib

    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 15, syms
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED_SYMBOLS)
    assert L.dma_abi_version() == 1


def test_plan_helper_matches_oracle(golden):
    from paper_2604_03950_b200 import _lib

    L = _lib.lib()
    buf = (ctypes.c_int64 * 4096)()
    cases, flat, offs = golden["plan_cases"], golden["plan_flat"], golden["plan_offs"]
    for i, (tm, tn, T, S, causal, lq, lk, qt) in enumerate(cases):
        n = L.dma_tile_plan(int(qt), int(lq), int(lk), int(tm), int(tn), int(T), int(S), int(causal), buf, 4096)
        assert list(buf[:n]) == list(flat[offs[i]:offs[i + 1]]), (i, cases[i])


def test_hpf_helper_matches_reference(golden):
    from paper_2604_03950_b200 import _lib

    L = _lib.lib()
    for c, want in zip(golden["plan_cases"][:150], golden["hpf"]):
        tm, tn, T, S, causal, lq, lk, _ = (int(v) for v in c)
        assert L.dma_high_precision_fraction(lq, lk, tm, tn, T, S, causal) == want
    for c, want in zip(golden["hpf_big_cases"], golden["hpf_big"]):
        lq, lk, tm, tn, T, S, causal = (int(v) for v in c)
        assert L.dma_high_precision_fraction(lq, lk, tm, tn, T, S, causal) == want


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_03950_b200 import quantize_dual

    with pytest.raises(RuntimeError, match="CUDA"):
        quantize_dual(np.zeros((4, 32)))
