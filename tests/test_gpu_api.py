"""GPU parity through the public API against fixtures of the REAL reference.

Every golden case is rebuilt from its stored input arrays, run through
``run_with_report(parse(src))`` on the B200, and checked for: the reference's
output format, bit-exact output structure (level pos/crd), values within the
north-star tolerance (per row: max |err| <= 1e-5 * max of the absolute-value
contraction), the reference's op counters (closed forms), and the dense path.
"""

import numpy as np
import pytest
import torch

import paper_2405_16883_b200 as st
from conftest import golden_names, load_golden
from helpers import abs_bound, golden_tensor
from oracle.restate import parity_gate

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.mark.parametrize("case", golden_names())
def test_golden_case(case):
    g = load_golden(case)
    meta = g["meta"]
    tensors = {n: golden_tensor(g, n) for n in meta["inputs"]}
    e = st.parse(meta["src"], tensors)
    out, counter, report = st.run_with_report(e, tile_size=meta["tile_size"], tiling=meta["tiling"])
    assert report["path"] == meta["path"]
    assert out.format.name() == meta["out_format"]
    # structure: every compressed level bit-exact
    for k, lv in enumerate(out.storage.levels):
        if hasattr(lv, "pos"):
            assert lv.pos.cpu().numpy().tolist() == g[f"out_l{k}_pos"].tolist(), f"level {k} pos"
            assert lv.crd.cpu().numpy().tolist() == g[f"out_l{k}_crd"].tolist(), f"level {k} crd"
    assert st.nnz(out) == len(g["out_vals"])
    got = st.to_dense(out)
    want = g["out_dense"]
    ok, worst = parity_gate(got, want, abs_bound(e, tensors), TOL)
    assert ok, f"{case}: worst error ratio {worst}"
    if meta["counters"] is not None:
        assert counter.as_dict() == meta["counters"], (counter.as_dict(), meta["counters"])
    if report["path"] == "sparse":
        assert report["schedule"]["loop_order"] == meta["loop_order"]
        assert report["variants"], "no kernel variant recorded"


def test_kat_values_exact():
    g = load_golden("kat_sddmm_worked")
    tensors = {n: golden_tensor(g, n) for n in g["meta"]["inputs"]}
    e = st.parse(g["meta"]["src"], tensors)
    t, c = st.execute(st.schedule(e))
    assert st.to_dense(t)[0, 1] == 44.0 and c.scalar_mults == 3
    A = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 0), 1.0), ((1, 1), 2.0)], name="A")
    x = st.from_dense([3.0, 4.0], name="x")
    t, c = st.execute(st.schedule(st.parse("y(i) = A(i,j) * x(j)", {"A": A, "x": x})))
    assert st.to_dense(t).tolist() == [3.0, 8.0] and c.scalar_mults == 2


def test_arithmetic_zeros_kept():
    M = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 0), 1.0)], name="M")
    Q = st.from_dense([[0.0, 0.0], [1.0, 1.0]], name="Q")
    K = st.from_dense([[1.0, 1.0], [1.0, 1.0]], name="K")
    t = st.run(st.parse("S(i,j) = M(i,j) * Q(i,d) * K(j,d)", {"M": M, "Q": Q, "K": K}))
    assert st.nnz(t) == 1 and st.to_dense(t)[0, 0] == 0.0


def test_rebinding():
    r = np.random.default_rng(0)
    from helpers import random_tensor

    A1 = random_tensor(r, (50, 40), "csr", 0.2, "A")
    A2 = random_tensor(r, (50, 40), "csr", 0.2, "A")
    B = st.from_dense(r.uniform(-1, 1, (40, 8)), name="B")
    e = st.parse("C(i,k) = A(i,j) * B(j,k)", {"A": A1, "B": B})
    s = st.tile(e, st.schedule(e), 64)
    t2, _ = st.execute(s, bindings={"A": A2})
    e2 = st.parse("C(i,k) = A(i,j) * B(j,k)", {"A": A2, "B": B})
    np.testing.assert_allclose(st.to_dense(t2), st.eval_dense(e2), rtol=0, atol=1e-5)
    with pytest.raises(st.ShapeError):
        st.execute(s, bindings={"A": st.convert(A1, st.dcsr(50, 40))})


def test_expressions_without_a_kernel_run_on_the_device_walker():
    """No dedicated kernel -> the device loop-nest walker (generic.py), never the CPU."""
    r = np.random.default_rng(1)
    from helpers import random_tensor

    A = random_tensor(r, (6, 6), "csr", 0.3, "A")
    B = random_tensor(r, (6, 6), "csr", 0.3, "B")
    D = random_tensor(r, (6, 6), "csr", 0.3, "D")
    Ad = random_tensor(r, (6, 6), "dcsr", 0.3, "Ad")
    Bd = st.from_dense(r.uniform(-1, 1, (6, 4)), name="Bd")
    cases = [
        ("C(i,j) = A(i,j) * B(i,j) * D(i,j)", {"A": A, "B": B, "D": D}, None),   # three sparse factors
        ("C(i,j) = A(i,j) + B(i,j) + D(i,j)", {"A": A, "B": B, "D": D}, None),   # three sparse terms
        ("C(i,k) = Ad(i,j) * B(j,k)", {"Ad": Ad, "B": B}, None),                 # DCSR x CSR SpGEMM
        ("C(i,k) = A(i,j) * Bd(j,k)", {"A": A, "Bd": Bd}, st.csr(6, 4)),         # forced CSR output
    ]
    for src, b, fmt in cases:
        e = st.parse(src, b)
        out, _, report = st.run_with_report(e, out_format=fmt)
        assert out.storage.values.is_cuda
        assert report["variants"] and report["variants"][0].startswith("generic:device-walk"), report
        assert out.format == (fmt or st.infer_format(e))
        np.testing.assert_allclose(st.to_dense(out), st.eval_dense(e), rtol=1e-6, atol=1e-6)


def test_walk_too_large_raises():
    n = 200_000
    x = st.from_arrays((n,), st.TensorFormat((n,), (0,), (st.LevelFormat.COMPRESSED,)),
                       np.arange(n)[:, None], np.ones(n), name="x", device="cuda")
    y = st.from_arrays((n,), st.TensorFormat((n,), (0,), (st.LevelFormat.COMPRESSED,)),
                       np.arange(n)[:, None], np.ones(n), name="y", device="cuda")
    with pytest.raises(st.UnsupportedExpressionError):  # 4e10 outer-product entries
        st.run(st.parse("G(i,j) = x(i) * y(j)", {"x": x, "y": y}))


def test_dense_dispatch_matches_hand_results():
    cases = [
        ("C(i,k) = A(i,j) * B(j,k)", {"A": [[1.0, 2.0], [3.0, 4.0]], "B": [[5.0, 6.0], [7.0, 8.0]]},
         [[19.0, 22.0], [43.0, 50.0]]),
        ("C(i,j) = A(i,j) + B(i,j)", {"A": [[1.0, 0.0], [0.0, 1.0]], "B": [[0.0, 2.0], [3.0, 0.0]]},
         [[1.0, 2.0], [3.0, 1.0]]),
        ("y(i) = A(i,j) * x(j)", {"A": [[2.0, 0.0], [1.0, 3.0]], "x": [1.0, 2.0]}, [2.0, 7.0]),
    ]
    for src, raw, expected in cases:
        b = {n: st.from_dense(np.asarray(v), name=n) for n, v in raw.items()}
        t, counter, report = st.run_with_report(st.parse(src, b))
        assert report["path"] == "dense" and counter is None
        assert np.array_equal(st.to_dense(t), np.asarray(expected))


def test_device_storage_and_convert():
    from helpers import random_tensor

    r = np.random.default_rng(5)
    t = random_tensor(r, (30, 20), "csr", 0.3, "T")
    assert t.storage.values.is_cuda
    d = st.to_dense(t)
    for name in ("csr", "csc", "dcsr", "coo", "dense"):
        c = st.convert(t, st.format_by_name(name, (30, 20)))
        assert c.storage.values.is_cuda
        assert np.array_equal(st.to_dense(c), d)


def test_torch_dispatch():
    from helpers import random_tensor

    r = np.random.default_rng(7)
    A = random_tensor(r, (40, 30), "csr", 0.2, "A")
    B = torch.randn(30, 16, device="cuda")
    want = torch.from_numpy(st.to_dense(A)).cuda().float() @ B
    for got in (torch.mm(A, B), torch.matmul(A, B), A @ B, torch.einsum("ij,jk->ik", A, B),
                torch.sparse.mm(A, B)):
        assert isinstance(got, torch.Tensor) and got.is_cuda
        torch.testing.assert_close(got, want, rtol=1e-5, atol=1e-5)
    x = torch.randn(30, device="cuda")
    torch.testing.assert_close(A @ x, want.new_tensor(st.to_dense(A)).float() @ x, rtol=1e-5, atol=1e-5)
    Ac = random_tensor(r, (40, 30), "coo", 0.2, "Ac")
    torch.testing.assert_close(torch.mm(Ac, B), torch.from_numpy(st.to_dense(Ac)).cuda().float() @ B,
                               rtol=1e-5, atol=1e-5)
    # dense-only torch calls are untouched
    D = torch.randn(3, 3, device="cuda")
    assert torch.equal(torch.mm(D, D), D @ D)
