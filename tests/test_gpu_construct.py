"""Device-side construction (§8(f)-1): exact duplicate folding on the GPU reproduces the
reference's per-coordinate ``math.fsum`` (`/root/reference/pkg/src/sparsetc/tensor.py:238-241`)
bit for bit, including its exceptions, and device construction matches host construction."""

import math

import numpy as np
import pytest
import torch

import paper_2405_16883_b200 as st
from paper_2405_16883_b200.tensor import _fold_duplicates

pytestmark = pytest.mark.gpu


def _groups(rng, n_groups):
    """Adversarial float64 groups: cancellation, huge + tiny, ties at half an ulp, subnormals."""
    groups = []
    for g in range(n_groups):
        kind = g % 6
        m = int(rng.integers(2, 40))
        if kind == 0:
            x = rng.standard_normal(m) * 10.0 ** rng.integers(-300, 300, m)
        elif kind == 1:
            big = rng.standard_normal() * 1e16
            x = np.concatenate([[big, -big], rng.standard_normal(m)])
        elif kind == 2:
            x = np.concatenate([[1.0, 2.0 ** -53, 2.0 ** -106], rng.choice([1.0, -1.0], m) * 2.0 ** -60])
        elif kind == 3:
            x = rng.uniform(-1, 1, m) * 5e-324 * rng.integers(1, 1000, m)
        elif kind == 4:
            x = np.repeat(rng.standard_normal(), m) * np.where(np.arange(m) % 2, -1.0, 1.0)
        else:
            x = rng.uniform(-1, 1, m).astype(np.float32).astype(np.float64)
        groups.append(rng.permutation(x))
    return groups


def test_device_fsum_matches_math_fsum_bitwise():
    rng = np.random.default_rng(2024)
    groups = _groups(rng, 3000)
    vals = np.concatenate(groups)
    keys = np.repeat(np.arange(len(groups)), [len(g) for g in groups])
    cs = torch.from_numpy(keys).cuda()[:, None]
    same = cs[1:, 0] == cs[:-1, 0]
    _, out = _fold_duplicates(cs, torch.from_numpy(vals).cuda(), same)
    want = np.array([math.fsum(g) for g in groups])
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


@pytest.mark.parametrize("values,want", [
    ([1.0, float("nan")], "nan"),
    ([float("inf"), 1.0, 2.0], float("inf")),
    ([float("-inf"), float("-inf")], float("-inf")),
])
def test_device_fsum_special_values(values, want):
    cs = torch.zeros((len(values), 1), dtype=torch.long, device="cuda")
    _, out = _fold_duplicates(cs, torch.tensor(values, dtype=torch.float64, device="cuda"),
                              torch.ones(len(values) - 1, dtype=torch.bool, device="cuda"))
    ref = math.fsum(values)
    if want == "nan":
        assert math.isnan(out.item()) and math.isnan(ref)
    else:
        assert out.item() == want == ref


def test_device_fsum_raises_like_fsum():
    cs = torch.zeros((2, 1), dtype=torch.long, device="cuda")
    one = torch.ones(1, dtype=torch.bool, device="cuda")
    with pytest.raises(ValueError):
        math.fsum([float("inf"), float("-inf")])
    with pytest.raises(ValueError):
        _fold_duplicates(cs, torch.tensor([float("inf"), float("-inf")], dtype=torch.float64, device="cuda"), one)
    with pytest.raises(OverflowError):
        math.fsum([1.7e308, 1.7e308])
    with pytest.raises(OverflowError):
        _fold_duplicates(cs, torch.tensor([1.7e308, 1.7e308], dtype=torch.float64, device="cuda"), one)


@pytest.mark.parametrize("fmt_name", ["csr", "csc", "dcsr", "coo", "dense"])
def test_build_from_entries_device_equals_host(fmt_name):
    rng = np.random.default_rng(7)
    shape = (40, 30)
    n = 2000  # ~1.7 entries per coordinate: many duplicate groups
    coords = np.stack([rng.integers(0, 40, n), rng.integers(0, 30, n)], 1)
    vals = rng.standard_normal(n) * 10.0 ** rng.integers(-8, 8, n)
    entries = [(tuple(c), float(v)) for c, v in zip(coords, vals)]
    fmt = st.format_by_name(fmt_name, shape)
    d = st.build_from_entries(shape, fmt, entries, name="T", device="cuda")
    h = st.build_from_entries(shape, fmt, entries, name="T", device="cpu")
    assert d.storage.values.is_cuda
    assert torch.equal(d.storage.values.cpu(), h.storage.values)
    for a, b in zip(d.storage.levels, h.storage.levels):
        for attr in ("pos", "crd"):
            if hasattr(a, attr):
                assert torch.equal(getattr(a, attr).cpu(), getattr(b, attr))


def test_from_arrays_at_cfg5_scale_on_device():
    """The 10 M raw cfg5 draws (with repeats) folded on the device, checked against a
    host float64 reference on a sample of the repeated coordinates."""
    from paper_2405_16883_b200 import synthetic

    rng = synthetic.tensor_rng("T")
    i, j, k = (synthetic.truncated_zipf(rng, 10_000_000, 20000, 1.1) for _ in range(3))
    vals = np.random.default_rng(3).uniform(0, 1, len(i))
    coords = np.stack([i, j, k], 1)
    fmt = st.TensorFormat((20000,) * 3, (0, 1, 2), (st.LevelFormat.COORDINATE,) * 3)
    T = st.from_arrays((20000,) * 3, fmt, torch.from_numpy(coords).cuda(), torch.from_numpy(vals).cuda(),
                       name="T", device="cuda")
    key = (i * 20000 + j) * 20000 + k
    uk, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
    assert st.nnz(T) == len(uk)
    sums = np.zeros(len(uk))
    np.add.at(sums, inv, vals)
    got = T.storage.values.cpu().numpy()
    rep = np.flatnonzero(cnt > 1)[:20000]
    assert np.allclose(got[rep], sums[rep].astype(np.float32), rtol=1e-6, atol=0)
