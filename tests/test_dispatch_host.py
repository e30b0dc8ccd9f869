"""torch interception without a GPU: unsupported torch functions on a declared sparse tensor
raise instead of silently densifying it; all-dense tensors fall through to torch."""

import numpy as np
import pytest
import torch

import paper_2405_16883_b200 as st

from helpers import random_tensor


def test_unhandled_torch_function_on_sparse_raises():
    A = random_tensor(np.random.default_rng(1), (8, 6), "csr", 0.3, "A")
    with pytest.raises(TypeError, match="no sparse kernel"):
        torch.add(A, 1.0)
    with pytest.raises(TypeError):
        torch.sum(A)


def test_dense_tensor_falls_through():
    D = st.from_dense(np.arange(6.0).reshape(2, 3), name="D")
    assert torch.equal(torch.sum(D), torch.tensor(15.0))
