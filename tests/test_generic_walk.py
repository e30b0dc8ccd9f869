"""The device loop-nest walker (generic.py) against the real reference engine.

Fixtures: tests/golden/walk/generic_walk.npz and generic_walk_tiled.npz (one index extent in
[65, 140] and the plan tiles it, so tiled loops run several 64-wide blocks), made by
tests/golden/make_generic_golden.py (the reference's run_with_report on its own
random-expression strategy, plus hand cases). The CPU tests run the walker on CPU-resident
buffers (it is device-agnostic torch; the product path requires CUDA); the GPU test goes
through the public API, where expressions without a dedicated kernel dispatch to the walker
on the device. Structure (format, pos/crd) must be bit-identical; values within float32
rounding of the reference's float64 result (the walker sums in float64 and rounds once);
the OpCounter equal to the reference interpreter's (walk_count.py).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import paper_2405_16883_b200 as st
from paper_2405_16883_b200.engine import OpCounter
from paper_2405_16883_b200.generic import execute_generic
from paper_2405_16883_b200.tiling import tile

DIR = Path(__file__).resolve().parent / "golden" / "walk"
FIX = {name: np.load(DIR / f"{name}.npz") for name in ("generic_walk", "generic_walk_tiled")}
CASES = {name: [str(c) for c in z["cases"]] for name, z in FIX.items()}
LV = {"dense": st.LevelFormat.DENSE, "compressed": st.LevelFormat.COMPRESSED,
      "coordinate": st.LevelFormat.COORDINATE}


def _fmt(z, p):
    shape = tuple(int(x) for x in z[p + "_shape"])
    return st.TensorFormat(shape, tuple(int(x) for x in z[p + "_modes"]), tuple(LV[str(k)] for k in z[p + "_levels"]))


def _fields(f, i):
    parts = [s.strip() for s in CASES[f][i].split("|")]
    return parts[0], parts[1], parts[2], (parts[3] if len(parts) > 3 else None)


def _case(f, i, device):
    z = FIX[f]
    src, names, path, _ = _fields(f, i)
    b = {}
    for n in names.split(","):
        p = f"c{i}_{n}"
        fmt = _fmt(z, p)
        b[n] = st.from_arrays(fmt.shape, fmt, z[p + "_coords"], z[p + "_vals"], name=n, device=device,
                              duplicates="error")
    return st.parse(src, b), path


def _check(f, i, out, tol_abs=None):
    z = FIX[f]
    q = f"c{i}_out"
    want_fmt = _fmt(z, q)
    assert out.format == want_fmt, (CASES[f][i], out.format, want_fmt)
    for k, lv in enumerate(out.storage.levels):
        if f"{q}_l{k}_pos" in z:
            assert np.array_equal(lv.pos.cpu().numpy().astype(np.int64), z[f"{q}_l{k}_pos"]), (CASES[f][i], k)
        if f"{q}_l{k}_crd" in z:
            assert np.array_equal(lv.crd.cpu().numpy().astype(np.int64), z[f"{q}_l{k}_crd"]), (CASES[f][i], k)
    want = z[q + "_vals"]
    got = out.storage.values.cpu().numpy().astype(np.float64)
    assert got.shape == want.shape, CASES[f][i]
    if tol_abs is None:  # the walker: float64 sums, one rounding to float32
        assert np.allclose(got, want, rtol=2e-7, atol=1e-12), (CASES[f][i], np.abs(got - want).max())
    else:                # a float32 kernel: the north-star gate against the |operand| contraction
        assert np.all(np.abs(got - want) <= tol_abs), (CASES[f][i], np.abs(got - want).max(), tol_abs)


def _out_format(f, i, e):
    name = _fields(f, i)[3]
    return None if name is None else st.format_by_name(name, e.output_shape)


ALL = [(f, i) for f in FIX for i in range(len(CASES[f]))]
SPARSE_CASES = [(f, i) for f, i in ALL if _fields(f, i)[2] == "sparse"]
COUNTED = [(f, i) for f, i in ALL if f"c{i}_counters" in FIX[f].files]


def _walk(f, i):
    e, _ = _case(f, i, "cpu")
    fmt = _out_format(f, i, e) or st.infer_format(e)
    sched = tile(e, st.schedule(e, fmt), 64)
    tensor_of = {id(a): a.tensor for a in e.accesses}
    cnt = OpCounter()
    return e, execute_generic(sched, tensor_of, fmt, cnt), cnt


def test_fixture_covers_the_random_strategy():
    assert len(CASES["generic_walk"]) >= 170 and len(CASES["generic_walk_tiled"]) >= 80
    assert len(SPARSE_CASES) >= 150 and len(COUNTED) >= 220


@pytest.mark.parametrize("f,i", SPARSE_CASES)
def test_walker_matches_reference_on_cpu_buffers(f, i):
    e, out, _ = _walk(f, i)
    _check(f, i, out)
    # eval_dense (public API) agrees with the reference's output, broadcast terms included
    np.testing.assert_allclose(st.to_dense(out), st.eval_dense(e), rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("f,i", COUNTED)
def test_walker_counters_equal_the_reference_interpreter(f, i):
    """The walker's OpCounter is the reference interpreter's exact count (engine.py:51-68)
    for every expression it runs: intersections in the reference's seek order, tile blocks,
    vectorised dense tails, union outer loops of sparse outputs."""
    _, _, cnt = _walk(f, i)
    want = [int(x) for x in FIX[f][f"c{i}_counters"]]
    assert [cnt.scalar_mults, cnt.scalar_adds, cnt.iterator_advances] == want, (CASES[f][i], want)


@pytest.mark.gpu
@pytest.mark.parametrize("f,i", ALL)
def test_public_api_matches_reference_on_device(f, i):
    from helpers import abs_bound

    e, _ = _case(f, i, "cuda")
    out, cnt, report = st.run_with_report(e, out_format=_out_format(f, i, e))
    kernel = not (report["variants"] and report["variants"][0].startswith("generic"))
    tensors = {a.tensor.name: a.tensor for a in e.accesses}
    _check(f, i, out, 1e-5 * float(np.max(abs_bound(e, tensors), initial=0.0)) if kernel else None)
    key = f"c{i}_counters"
    if key in FIX[f].files:  # kernels (closed forms) and the walker (walk_count) alike
        assert [cnt.scalar_mults, cnt.scalar_adds, cnt.iterator_advances] == [int(x) for x in FIX[f][key]], \
            (CASES[f][i], report["variants"])
