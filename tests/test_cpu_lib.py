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
    assert L.dma_abi_version() == _lib.ABI_VERSION == 2


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


def test_decode_abi_validation_on_host():
    """dma_decode_* argument checks run on the host before any CUDA call (include/dma.h):
    workspace sizing for valid shapes, DMA_EINVAL / DMA_EUNSUPPORTED with a message otherwise."""
    from paper_2604_03950_b200 import _lib
    from paper_2604_03950_b200.decode import DecodeArgs, _bind

    L = _bind()

    def args(**kw):
        a = DecodeArgs()
        base = dict(v_dtype=_lib.DT_BF16, out_dtype=_lib.DT_F32, batch=2, heads=8, kv_heads=2, n_q=1,
                    capacity=1024, pos=700, head_dim=128, v_dim=128, tile_m=128, tile_n=128, diag_window=128,
                    sink_window=128, low_format=_lib.FMT_NVFP4, high_format=_lib.FMT_MXFP8_E4M3,
                    granularity=_lib.GRAN_TOKEN)
        base.update(kw)
        for k, v in base.items():
            setattr(a, k, v)
        return a

    ws = L.dma_decode_workspace_bytes(args())
    rows = 2 * 8 * 1
    assert ws >= rows * 128 * 4 and ws % 8 == 0
    assert L.dma_decode_workspace_bytes(args(n_q=4)) > ws  # more query rows, more partials
    bad = {
        "capacity": (dict(capacity=1000), _lib.DMA_EINVAL, "multiple of 32"),
        "overflow": (dict(pos=1024), _lib.DMA_EINVAL, "capacity"),
        "gqa": (dict(heads=7), _lib.DMA_EINVAL, "kv_heads"),
        "gran": (dict(granularity=_lib.GRAN_TENSOR), _lib.DMA_EUNSUPPORTED, "TOKEN"),
        "dim": (dict(head_dim=96), _lib.DMA_EUNSUPPORTED, "64 or 128"),
        "tile": (dict(tile_n=48), _lib.DMA_EUNSUPPORTED, "multiple of 32"),
        "high": (dict(high_format=_lib.FMT_NVFP4), _lib.DMA_EUNSUPPORTED, "MXFP8"),
        "vdtype": (dict(v_dtype=_lib.DT_F32), _lib.DMA_EUNSUPPORTED, "bf16"),
    }
    for name, (kw, rc, msg) in bad.items():
        a = args(**kw)
        assert L.dma_decode_workspace_bytes(a) == 0, name
        assert L.dma_decode_attention(a, None) == rc, name
        assert msg in L.dma_last_error().decode(), (name, L.dma_last_error())
    # valid shape but no operand pointers: rejected before any launch
    assert L.dma_decode_attention(args(), None) == _lib.DMA_EINVAL
    assert "pointer" in L.dma_last_error().decode()


def test_attention_abi_validation_on_host():
    """dma_attention_supported / _workspace_bytes: the host-side coverage rules of the
    sm_100a kernels (include/dma.h), no GPU needed."""
    from paper_2604_03950_b200 import _lib

    L = _lib.lib()

    def args(**kw):
        a = _lib.DmaAttnArgs()
        base = dict(in_dtype=_lib.DT_BF16, out_dtype=_lib.DT_BF16, batch=1, heads=32, kv_heads=8, len_q=8192,
                    len_k=8192, head_dim=128, v_dim=128, tile_m=128, tile_n=128, diag_window=128,
                    sink_window=128, causal=1, low_format=_lib.FMT_MXFP4, high_format=_lib.FMT_MXFP8_E4M3,
                    granularity=_lib.GRAN_TOKEN, pv_mode=_lib.PV_MXFP8, prescale=1.0)
        base.update(kw)
        for k, v in base.items():
            setattr(a, k, v)
        return a

    assert L.dma_attention_supported(args()) == 0
    ws = L.dma_attention_workspace_bytes(args())
    # phase-1 operands of Q (32 heads) and K/V (8 heads) at 8192 x 128 must fit
    assert ws > (32 + 8) * 8192 * 128 * (1 + 0.5) + 8 * 8192 * 128
    for kw in (dict(tile_m=64, tile_n=64), dict(v_dim=64), dict(head_dim=64, v_dim=64),
               dict(granularity=_lib.GRAN_BLOCK), dict(low_format=_lib.FMT_NONE, high_format=_lib.FMT_NONE),
               dict(causal=0, len_k=5000), dict(pv_mode=_lib.PV_BF16)):
        assert L.dma_attention_supported(args(**kw)) == 0, kw
    for kw, rc in ((dict(tile_n=32), _lib.DMA_EUNSUPPORTED), (dict(head_dim=96, v_dim=96), _lib.DMA_EUNSUPPORTED),
                   (dict(len_k=4096), _lib.DMA_EINVAL), (dict(heads=30), _lib.DMA_EINVAL),
                   (dict(diag_window=100), _lib.DMA_EINVAL)):
        assert L.dma_attention_supported(args(**kw)) == rc, kw
        assert L.dma_last_error()


def test_kv_split_policy_host_only():
    """dma_attention_kv_split / dma_attention_set_kv_split are host logic (no GPU needed):
    small problems split, c3 does not, the per-call field and the global mode override."""
    import paper_2604_03950_b200 as D
    from paper_2604_03950_b200 import _lib

    L = _lib.lib()
    c = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=D.MXFP4)
    ks = D.attention.kv_split_count
    prev = L.dma_attention_set_kv_split(-1)
    try:
        assert ks((1, 1, 1024, 64), (1, 1, 1024, 64), (1, 1, 1024, 64), c) > 1
        assert ks((1, 32, 32768, 128), (1, 32, 32768, 128), (1, 32, 32768, 128), c) == 1
        L.dma_attention_set_kv_split(0)
        assert ks((1, 1, 1024, 64), (1, 1, 1024, 64), (1, 1, 1024, 64), c) == 1
        L.dma_attention_set_kv_split(3)
        assert ks((1, 1, 1024, 64), (1, 1, 1024, 64), (1, 1, 1024, 64), c) == 3
        assert ks((1, 1, 200, 64), (1, 1, 200, 64), (1, 1, 200, 64), c) == 2  # capped by the plan length
    finally:
        L.dma_attention_set_kv_split(prev)
