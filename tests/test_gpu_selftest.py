"""GPU: one-tile tcgen05 block-scaled MMA self-test against a numpy decode.

Validates the UMMA descriptor / swizzle / scale-factor-atom / A-from-TMEM
conventions the DMA kernel is built on."""

import numpy as np
import pytest

from oracle import mx_oracle as O

pytestmark = pytest.mark.gpu

E2M1_TAB = np.array([0, .5, 1, 1.5, 2, 3, 4, 6, -0., -.5, -1, -1.5, -2, -3, -4, -6])


def _fp8_codes(rng, shape):
    c = rng.integers(0, 256, size=shape).astype(np.uint8)
    c[(c & 0x7F) == 0x7F] = 0x10  # no NaN
    return c


def _e4m3_tab():
    return O.decode_fp8(np.arange(256), O.E4M3)


def _unpack(p, K):
    out = np.empty((p.shape[0], K), dtype=np.int64)
    out[:, 0::2] = p & 0xF
    out[:, 1::2] = p >> 4
    return out


def run(kind, K, a, b, sfa, sfb):
    import torch

    from paper_2604_03950_b200 import _lib

    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    ta, tb, tsa, tsb = dev(a), dev(b), dev(sfa), dev(sfb)
    d = torch.zeros((128, 128), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().dma_selftest_mma(kind, K, ta.data_ptr(), tb.data_ptr(), tsa.data_ptr(),
                                           tsb.data_ptr(), d.data_ptr(), _lib.stream_ptr()), "selftest")
    torch.cuda.synchronize()
    return d.cpu().numpy().astype(np.float64)


def close(got, ref, absref):
    err = np.abs(got - ref)
    tol = 2e-6 * absref + 1e-30
    bad = err > tol
    assert not bad.any(), f"{bad.sum()} mismatches; max err {err.max()} ; sample got {got[0, :4]} ref {ref[0, :4]}"


@pytest.mark.parametrize("K", [64, 128])
@pytest.mark.parametrize("e5", [False, True])
def test_mxf8(K, e5):
    rng = np.random.default_rng(K + e5)
    a, b = _fp8_codes(rng, (128, K)), _fp8_codes(rng, (128, K))
    if e5:
        a[(a & 0x7C) == 0x7C] = 0x10
        b[(b & 0x7C) == 0x7C] = 0x10
    sfa = rng.integers(120, 134, size=(128, K // 32)).astype(np.uint8)
    sfb = rng.integers(120, 134, size=(128, K // 32)).astype(np.uint8)
    tab = O.decode_fp8(np.arange(256), O.E5M2 if e5 else O.E4M3)
    A = tab[a] * np.repeat(np.exp2(sfa.astype(float) - 127), 32, axis=1)
    B = tab[b] * np.repeat(np.exp2(sfb.astype(float) - 127), 32, axis=1)
    got = run(5 if e5 else 0, K, a, b, sfa, sfb)
    close(got, A @ B.T, np.abs(A) @ np.abs(B).T)


@pytest.mark.parametrize("K", [64, 128])
def test_nvf4(K):
    rng = np.random.default_rng(10 + K)
    a = rng.integers(0, 256, size=(128, K // 2)).astype(np.uint8)
    b = rng.integers(0, 256, size=(128, K // 2)).astype(np.uint8)
    sfa = rng.integers(0x28, 0x48, size=(128, K // 16)).astype(np.uint8)
    sfb = rng.integers(0x28, 0x48, size=(128, K // 16)).astype(np.uint8)
    tab = _e4m3_tab()
    A = E2M1_TAB[_unpack(a, K)] * np.repeat(tab[sfa], 16, axis=1)
    B = E2M1_TAB[_unpack(b, K)] * np.repeat(tab[sfb], 16, axis=1)
    got = run(1, K, a, b, sfa, sfb)
    close(got, A @ B.T, np.abs(A) @ np.abs(B).T)


@pytest.mark.parametrize("K", [64, 128])
def test_mxf4(K):
    rng = np.random.default_rng(20 + K)
    a = rng.integers(0, 256, size=(128, K // 2)).astype(np.uint8)
    b = rng.integers(0, 256, size=(128, K // 2)).astype(np.uint8)
    sfa = rng.integers(120, 134, size=(128, K // 32)).astype(np.uint8)
    sfb = rng.integers(120, 134, size=(128, K // 32)).astype(np.uint8)
    A = E2M1_TAB[_unpack(a, K)] * np.repeat(np.exp2(sfa.astype(float) - 127), 32, axis=1)
    B = E2M1_TAB[_unpack(b, K)] * np.repeat(np.exp2(sfb.astype(float) - 127), 32, axis=1)
    got = run(2, K, a, b, sfa, sfb)
    close(got, A @ B.T, np.abs(A) @ np.abs(B).T)


@pytest.mark.parametrize("K", [64, 128])
def test_pv_fp8_tmem_a(K):
    rng = np.random.default_rng(30 + K)
    p = _fp8_codes(rng, (128, K)) & 0x7F  # P >= 0
    v = _fp8_codes(rng, (K, 128))
    sfp = rng.integers(120, 134, size=(128, K // 32)).astype(np.uint8)
    sfv = rng.integers(120, 134, size=(128, K // 32)).astype(np.uint8)  # [n, key block]
    tab = _e4m3_tab()
    P = tab[p] * np.repeat(np.exp2(sfp.astype(float) - 127), 32, axis=1)
    V = tab[v] * np.repeat(np.exp2(sfv.astype(float) - 127), 32, axis=1).T
    got = run(3, K, p, v, sfp, sfv)
    close(got, P @ V, np.abs(P) @ np.abs(V))


@pytest.mark.parametrize("K", [64, 128])
def test_pv_bf16_tmem_a(K):
    import torch

    rng = np.random.default_rng(40 + K)
    P = torch.from_numpy(rng.standard_normal((128, K))).to(torch.bfloat16)
    V = torch.from_numpy(rng.standard_normal((K, 128))).to(torch.bfloat16)
    pa = P.view(torch.uint8).numpy().reshape(128, 2 * K)
    vb = V.view(torch.uint8).numpy().reshape(K, 256)
    dummy = np.zeros((128, 4), np.uint8)
    got = run(4, K, pa, vb, dummy, dummy)
    Pf, Vf = P.double().numpy(), V.double().numpy()
    close(got, Pf @ Vf, np.abs(Pf) @ np.abs(Vf))
