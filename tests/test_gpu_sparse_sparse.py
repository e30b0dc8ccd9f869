"""Sparse x sparse on the B200: SpGEMM and CSR union / product.

Structure (rowptr, colidx) must equal the float64 oracle's bit for bit (the
reference keeps every touched coordinate, zeros included); values pass the
north-star gate: per output row max |gpu - oracle| <= 1e-5 * max of the row's
absolute-value result (|A| @ |B|, |A| + |B|, |A| .* |B|).
"""

import numpy as np
import pytest
import torch

import paper_2405_16883_b200 as st
from oracle import restate
from oracle.restate import parity_gate
from paper_2405_16883_b200 import ops

pytestmark = pytest.mark.gpu

TOL = 1e-5


def make_csr(rng, m, n, lens, zero_frac=0.0):
    lens = np.minimum(np.asarray(lens, dtype=np.int64), n)
    rp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    ci = (np.concatenate([np.sort(rng.choice(n, int(L), replace=False)) for L in lens])
          if m else np.zeros(0)).astype(np.int64)
    v = rng.uniform(-1, 1, rp[-1]).astype(np.float32)
    if zero_frac:
        v[rng.random(len(v)) < zero_frac] = 0.0
    return rp, ci, v


def dev(rp, ci, v):
    return (torch.from_numpy(rp).int().cuda(), torch.from_numpy(ci).int().cuda(),
            torch.from_numpy(v).float().cuda())


def dense_of(rp, ci, v, shape):
    out = np.zeros(shape)
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    out[rows, ci] = v
    return out


def check(res, want, bound_dense, shape):
    rp, ci, v = want
    assert res.rowptr.cpu().numpy().tolist() == np.asarray(rp).tolist()
    assert res.colidx.cpu().numpy().tolist() == np.asarray(ci).tolist()
    got = dense_of(rp, ci, res.vals.cpu().numpy().astype(np.float64), shape)
    ok, worst = parity_gate(got, dense_of(rp, ci, v, shape), bound_dense, TOL)
    assert ok, f"worst error ratio {worst}"


SPGEMM = {
    "uniform": lambda r: ((300, 200, r.integers(0, 12, 300)), (200, 250, r.integers(0, 12, 200))),
    "empty_rows": lambda r: ((64, 50, np.where(np.arange(64) % 3 == 0, 0, 5)),
                             (50, 70, np.where(np.arange(50) % 4 == 1, 0, 6))),
    "dense_rows": lambda r: ((40, 300, np.where(np.arange(40) == 7, 300, r.integers(0, 5, 40))),
                             (300, 90, np.where(np.arange(300) % 50 == 0, 90, r.integers(0, 3, 300)))),
    "all_empty": lambda r: ((17, 9, np.zeros(17, dtype=np.int64)), (9, 11, r.integers(0, 5, 9))),
    "no_products": lambda r: ((10, 6, np.full(10, 2)), (6, 8, np.zeros(6, dtype=np.int64))),
    "single": lambda r: ((1, 1, [1]), (1, 1, [1])),
    "power_law": lambda r: ((2000, 2000, np.minimum((2000 / (np.arange(2000) + 1)) ** 0.8 + 1, 2000).astype(int)),
                            (2000, 2000, r.integers(0, 8, 2000))),
    # B wider than the SMEM window (6144 columns): expand-sort-compress path
    "wide_esc": lambda r: ((120, 300, r.integers(0, 25, 120)), (300, 20000, r.integers(0, 40, 300))),
    "wide_esc_dense_row": lambda r: ((30, 100, np.where(np.arange(30) == 3, 100, r.integers(0, 4, 30))),
                                     (100, 9000, np.where(np.arange(100) == 10, 9000, r.integers(0, 30, 100)))),
    "wide_esc_no_products": lambda r: ((10, 6, np.full(10, 2)), (6, 7000, np.zeros(6, dtype=np.int64))),
}


@pytest.mark.parametrize("struct", list(SPGEMM))
def test_spgemm(struct):
    rng = np.random.default_rng(abs(hash(struct)) % 2**32)
    (m, n, la), (n2, p, lb) = SPGEMM[struct](rng)
    assert n == n2
    A = make_csr(rng, m, n, la, zero_frac=0.05)
    B = make_csr(rng, n, p, lb)
    want = restate.spgemm_csr(*A, *B)
    res = ops.spgemm_csr(*dev(*A), *dev(*B), p)
    assert res.products == int(np.diff(B[0])[A[1]].sum())
    bound = dense_of(*A, (m, n)).__abs__() @ dense_of(*B, (n, p)).__abs__()
    check(res, want, bound, (m, p))


def test_spgemm_deterministic():
    rng = np.random.default_rng(5)
    A = dev(*make_csr(rng, 500, 400, rng.integers(0, 20, 500)))
    B = dev(*make_csr(rng, 400, 300, rng.integers(0, 20, 400)))
    r1, r2 = ops.spgemm_csr(*A, *B, 300), ops.spgemm_csr(*A, *B, 300)
    assert torch.equal(r1.colidx, r2.colidx) and torch.equal(r1.vals, r2.vals)


EWISE = {
    "uniform": lambda r: (300, 200, r.integers(0, 40, 300), r.integers(0, 40, 300)),
    "disjoint_rows": lambda r: (50, 80, np.where(np.arange(50) % 2 == 0, 10, 0), np.where(np.arange(50) % 2, 10, 0)),
    "long_rows": lambda r: (8, 5000, [4000, 0, 77, 5000, 1, 2, 3000, 64], [3000, 5, 0, 5000, 1, 33, 3500, 64]),
    "all_empty": lambda r: (12, 7, np.zeros(12, dtype=np.int64), np.zeros(12, dtype=np.int64)),
    "one_empty": lambda r: (30, 40, r.integers(0, 9, 30), np.zeros(30, dtype=np.int64)),
}


@pytest.mark.parametrize("struct", list(EWISE))
@pytest.mark.parametrize("op", ["add", "mul"])
def test_csr_ewise(struct, op):
    rng = np.random.default_rng(abs(hash((struct, op))) % 2**32)
    m, n, la, lb = EWISE[struct](rng)
    A = make_csr(rng, m, n, la)
    B = make_csr(rng, m, n, lb)
    want = restate.csr_ewise(op, *A, *B)
    res = ops.csr_ewise(op, *dev(*A), *dev(*B))
    da, db = np.abs(dense_of(*A, (m, n))), np.abs(dense_of(*B, (m, n)))
    check(res, want, da + db if op == "add" else da * db, (m, n))


def test_ewise_values_follow_reference_order():
    # (0 + a) + b: a lone -0.0 becomes +0.0 in the workspace, like the reference's dict slot
    A = (np.array([0, 2]), np.array([0, 1]), np.array([-0.0, 1.5], dtype=np.float32))
    B = (np.array([0, 1]), np.array([1]), np.array([2.25], dtype=np.float32))
    res = ops.csr_ewise("add", *dev(*A), *dev(*B))
    v = res.vals.cpu().numpy()
    assert v.tolist() == [0.0, 3.75] and not np.signbit(v[0])


def test_engine_spgemm_and_ewise_through_api():
    rng = np.random.default_rng(11)
    A = st.from_dense((rng.random((30, 20)) < 0.2) * rng.uniform(-1, 1, (30, 20)), st.csr(30, 20), name="A")
    B = st.from_dense((rng.random((20, 25)) < 0.2) * rng.uniform(-1, 1, (20, 25)), st.csr(20, 25), name="B")
    A2 = st.from_dense((rng.random((30, 20)) < 0.3) * rng.uniform(-1, 1, (30, 20)), st.csr(30, 20), name="A2")
    for src, tensors, dense in [
        ("C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B}, lambda: st.to_dense(A) @ st.to_dense(B)),
        ("C(i,j) = A(i,j) + A2(i,j)", {"A": A, "A2": A2}, lambda: st.to_dense(A) + st.to_dense(A2)),
        ("C(i,j) = A(i,j) * A2(i,j)", {"A": A, "A2": A2}, lambda: st.to_dense(A) * st.to_dense(A2)),
    ]:
        e = st.parse(src, tensors)
        out, counter, report = st.run_with_report(e)
        assert report["out_format"] == "csr" and report["variants"]
        assert np.allclose(st.to_dense(out), dense(), atol=1e-5)


def test_non_csr_sparse_sparse_runs_on_the_device_walker():
    """COO x CSR has no SpGEMM kernel: the device loop-nest walker computes it."""
    rng = np.random.default_rng(12)
    A = st.from_dense((rng.random((10, 8)) < 0.3) * 1.0, st.coo(10, 8), name="A")
    B = st.from_dense((rng.random((8, 9)) < 0.3) * 1.0, st.csr(8, 9), name="B")
    e = st.parse("C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})
    out, _, report = st.run_with_report(e)
    assert report["variants"][0].startswith("generic:device-walk")
    assert out.format == st.infer_format(e)
    assert np.allclose(st.to_dense(out), st.to_dense(A) @ st.to_dense(B), atol=1e-6)
