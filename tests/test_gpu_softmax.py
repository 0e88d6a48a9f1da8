"""Tile-level softmax helpers (attention.py:83-106, 150-184) vs golden vectors frozen from the
live reference (tests/golden/make_softmax_golden.py)."""

import os

import numpy as np
import pytest

import paper_2604_03950_b200 as D
from paper_2604_03950_b200 import attention as DA

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "softmax_golden.npz"))
pytestmark = pytest.mark.gpu


def test_reference_names_exported():
    for name in ("OnlineSoftmaxState", "online_softmax_update", "apply_causal_mask"):
        assert getattr(DA, name) is getattr(D, name)


@pytest.mark.parametrize("ci", [0, 1, 2])
def test_online_softmax_chain(ci):
    rows, cols, d, base2 = (int(x) for x in G[f"c{ci}_meta"])
    st = D.OnlineSoftmaxState.fresh(rows, d)
    for t in range(4):
        st = D.online_softmax_update(st, G[f"c{ci}_t{t}_scores"], G[f"c{ci}_t{t}_v"], base2=bool(base2))
        m, l, o = st.numpy()
        np.testing.assert_array_equal(m, G[f"c{ci}_t{t}_m"])
        np.testing.assert_allclose(l, G[f"c{ci}_t{t}_l"], rtol=1e-13, atol=0)
        np.testing.assert_allclose(o, G[f"c{ci}_t{t}_o"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(st.normalized().cpu().numpy(), G[f"c{ci}_norm"], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("mi", [0, 1, 2, 3])
def test_apply_causal_mask(mi):
    qs, ks = (int(x) for x in G[f"mask{mi}_meta"])
    np.testing.assert_array_equal(D.apply_causal_mask(G[f"mask{mi}_in"], qs, ks), G[f"mask{mi}_out"])
    import torch

    t = D.apply_causal_mask(torch.from_numpy(G[f"mask{mi}_in"]).cuda(), qs, ks)
    assert isinstance(t, torch.Tensor) and t.is_cuda
    np.testing.assert_array_equal(t.cpu().numpy(), G[f"mask{mi}_out"])
