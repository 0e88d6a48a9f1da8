"""GPU: drop-in API robustness: operand validation at the raw-pointer
boundary, the reference's non-finite ValueError on the torch path (quantize.py:142-143),
and the lifetime of captured host-pipeline graphs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def D():
    import paper_2604_03950_b200 as m

    return m


def _cfg():
    d = D()
    return d.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=d.MXFP4)


def _qkv(B=1, H=2, KVH=2, N=256, d=64, seed=0, dtype=None, device="cuda"):
    import torch

    g = torch.Generator().manual_seed(seed)
    dt = dtype or torch.bfloat16
    mk = lambda h: torch.randn(B, h, N, d, generator=g).to(dt).to(device)  # noqa: E731
    return mk(H), mk(KVH), mk(KVH)


def test_prepare_rejects_strided_and_mixed_operands():
    import torch

    q, k, v = _qkv()
    fwd = D().DmaAttention(_cfg())
    # the standard model layout [B, L, H, D] viewed as [B, H, L, D] is not contiguous
    qt = q.transpose(1, 2).contiguous().transpose(1, 2)
    with pytest.raises(ValueError, match="contiguous"):
        fwd.prepare(qt, k, v)
    with pytest.raises(ValueError, match="dtypes differ"):
        fwd.prepare(q, k.float(), v)
    with pytest.raises(ValueError, match="out dtype"):
        fwd.prepare(q, k, v, out=torch.empty(q.shape, dtype=torch.float16, device="cuda"))
    with pytest.raises(ValueError, match="shape"):
        fwd.prepare(q, k, v, out=torch.empty((1, 2, 255, 64), dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(ValueError, match="CUDA"):
        fwd.prepare(q, k.cpu(), v)


def test_functional_api_accepts_strided_views():
    """dma_attention makes any layout contiguous: a transposed view gives the same output."""
    import torch

    q, k, v = _qkv(seed=1)
    want = D().dma_attention(q, k, v, _cfg())
    qv = q.transpose(1, 2).contiguous().transpose(1, 2)  # same values, strided
    got = D().dma_attention(qv, k, v, _cfg())
    assert torch.equal(got, want)


@pytest.mark.parametrize("where", ["q", "k"])
@pytest.mark.parametrize("bad", [float("nan"), float("inf")])
def test_nonfinite_query_key_raise(where, bad):
    """quantize.py:142-143: ValueError on NaN / Inf in Q or K (torch path, device flag)."""
    q, k, v = _qkv(seed=2)
    (q if where == "q" else k)[0, 1, 17, 5] = bad
    with pytest.raises(ValueError, match="non-finite"):
        D().dma_attention(q, k, v, _cfg())
    with pytest.raises(ValueError, match="non-finite"):
        D().mixed_precision_attention(q, k, v, _cfg())


def test_nonfinite_value_is_not_checked():
    """The reference only quantizes Q and K; V enters the float64 math as is (no error)."""
    q, k, v = _qkv(seed=3)
    v[0, 0, 3, 3] = float("nan")
    D().dma_attention(q, k, v, _cfg())  # no exception


def test_validate_off_is_asynchronous_and_flag_clears():
    """DmaAttention(validate=True) re-arms its flag every call: a clean call after a bad one passes."""
    q, k, v = _qkv(seed=4)
    fwd = D().DmaAttention(_cfg(), validate=True)
    k2 = k.clone()
    k2[0, 0, 0, 0] = float("nan")
    with pytest.raises(ValueError):
        fwd(q, k2, v)
    fwd(q, k, v)  # flag zeroed by the call itself
    D().DmaAttention(_cfg())(q, k2, v)  # validate=False: no check, no sync


def test_host_graph_cache_survives_pipe_eviction():
    """ADVICE (high): graphs captured for pinned host tensors must not outlive the device
    buffers they replay into.  Cycle three shapes (the pipe cache holds two), then
    re-run the first shape: it must equal a fresh device-side forward."""
    import torch

    fwd = D().DmaAttention(_cfg())
    sets = []
    for i, (B, H, KVH, N) in enumerate([(1, 4, 2, 512), (1, 4, 4, 384), (1, 2, 2, 640)]):
        q, k, v = _qkv(B, H, KVH, N, 64, seed=10 + i)
        host = tuple(t.cpu().pin_memory() for t in (q, k, v))
        sets.append(host + (torch.empty(B, H, N, 64, dtype=torch.bfloat16).pin_memory(),))
    for hq, hk, hv, ho in sets + sets[:1]:
        for _ in range(2):  # eager run + capture, then replay
            fwd.forward_host(hq, hk, hv, out=ho, chunk_kv_heads=1)
        torch.cuda.synchronize()
        ref = D().dma_attention(hq.cuda(), hk.cuda(), hv.cuda(), _cfg()).cpu()
        assert torch.equal(ho, ref), tuple(hq.shape)


def test_host_pipeline_pageable_inputs():
    """Non-pinned host tensors run the eager pipeline (copies from pageable memory are not
    captured into a graph) and give the device result."""
    import torch

    q, k, v = _qkv(1, 4, 2, 512, 64, seed=20)
    hq, hk, hv = q.cpu(), k.cpu(), v.cpu()
    fwd = D().DmaAttention(_cfg())
    for _ in range(2):
        out = fwd(hq, hk, hv)
    torch.cuda.synchronize()
    assert torch.equal(out, D().dma_attention(q, k, v, _cfg()).cpu())
    assert np.isfinite(out.float().numpy()).all()
