"""The device loop-nest walker (generic.py) against the real reference engine.

Fixtures: tests/golden/walk/generic_walk.npz, made by tests/golden/make_generic_golden.py
(the reference's run_with_report on its own random-expression strategy). The CPU test
runs the walker on CPU-resident buffers (it is device-agnostic torch; the product path
requires CUDA); the GPU test goes through the public API, where expressions without a
dedicated kernel dispatch to the walker on the device.
Structure (format, pos/crd) must be bit-identical; values within float32 rounding of
the reference's float64 result (the walker sums in float64 and rounds once).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2405_16883_b200 as st
from paper_2405_16883_b200.engine import OpCounter
from paper_2405_16883_b200.generic import execute_generic
from paper_2405_16883_b200.tiling import tile

FIX = Path(__file__).resolve().parent / "golden" / "walk" / "generic_walk.npz"
Z = np.load(FIX)
CASES = [str(c) for c in Z["cases"]]
LV = {"dense": st.LevelFormat.DENSE, "compressed": st.LevelFormat.COMPRESSED,
      "coordinate": st.LevelFormat.COORDINATE}


def _fmt(p):
    shape = tuple(int(x) for x in Z[p + "_shape"])
    return st.TensorFormat(shape, tuple(int(x) for x in Z[p + "_modes"]), tuple(LV[str(k)] for k in Z[p + "_levels"]))


def _fields(i):
    f = [s.strip() for s in CASES[i].split("|")]
    return f[0], f[1], f[2], (f[3] if len(f) > 3 else None)


def _case(i, device):
    src, names, path, _ = _fields(i)
    b = {}
    for n in names.split(","):
        p = f"c{i}_{n}"
        fmt = _fmt(p)
        b[n] = st.from_arrays(fmt.shape, fmt, Z[p + "_coords"], Z[p + "_vals"], name=n, device=device,
                              duplicates="error")
    return st.parse(src, b), path


def _check(i, out):
    q = f"c{i}_out"
    want_fmt = _fmt(q)
    assert out.format == want_fmt, (CASES[i], out.format, want_fmt)
    for k, lv in enumerate(out.storage.levels):
        if f"{q}_l{k}_pos" in Z:
            assert np.array_equal(lv.pos.cpu().numpy().astype(np.int64), Z[f"{q}_l{k}_pos"]), (CASES[i], k)
        if f"{q}_l{k}_crd" in Z:
            assert np.array_equal(lv.crd.cpu().numpy().astype(np.int64), Z[f"{q}_l{k}_crd"]), (CASES[i], k)
    want = Z[q + "_vals"]
    got = out.storage.values.cpu().numpy().astype(np.float64)
    assert got.shape == want.shape, CASES[i]
    assert np.allclose(got, want, rtol=2e-7, atol=1e-12), (CASES[i], np.abs(got - want).max())


SPARSE_CASES = [i for i in range(len(CASES)) if _fields(i)[2] == "sparse"]


def _out_format(i, e):
    name = _fields(i)[3]
    return None if name is None else st.format_by_name(name, e.output_shape)


def test_fixture_covers_the_random_strategy():
    assert len(CASES) >= 170 and len(SPARSE_CASES) >= 100


@pytest.mark.parametrize("i", SPARSE_CASES)
def test_walker_matches_reference_on_cpu_buffers(i):
    e, _ = _case(i, "cpu")
    fmt = _out_format(i, e) or st.infer_format(e)
    sched = tile(e, st.schedule(e, fmt), 64)
    tensor_of = {id(a): a.tensor for a in e.accesses}
    out = execute_generic(sched, tensor_of, fmt, OpCounter())
    _check(i, out)
    # eval_dense (public API) agrees with the reference's output, broadcast terms included
    np.testing.assert_allclose(st.to_dense(out), st.eval_dense(e), rtol=1e-6, atol=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(CASES)))
def test_public_api_matches_reference_on_device(i):
    e, _ = _case(i, "cuda")
    out, _, report = st.run_with_report(e, out_format=_out_format(i, e))
    _check(i, out)
