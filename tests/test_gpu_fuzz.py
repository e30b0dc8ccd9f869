"""Differential fuzz of the device path on the B200 (the reference's strategy,
tests/test_acceptance.py:101-116: random inputs checked against the dense evaluator).

1. Hot-path expressions with random extents, densities, formats, index names, operand
   order and operand spellings (SpMM / SpMV with or without a dense addend, transposed dense
   operands, SDDMM, MTTKRP, SpGEMM, CSR union / product) must run on a device kernel, come
   back in the inferred format and match the float64 dense evaluation within the north-star gate.
2. Fully random expressions (the reference's generator) all run on the device — a
   dedicated kernel or the device loop-nest walker (generic.py) — and match.
"""

import numpy as np
import pytest

import paper_2405_16883_b200 as st
from helpers import abs_bound, random_expression, random_tensor
from oracle.restate import parity_gate

pytestmark = pytest.mark.gpu

SPARSE = ("csr", "coo", "dcsr", "csc")


def _dense(rng, shape, name):
    return st.from_dense(rng.uniform(-1, 1, shape).astype(np.float32).astype(np.float64), name=name)


def _hot_path_case(rng, cap=40):
    names = list("ijklmnpq")
    rng.shuffle(names)
    i, j, k = names[:3]
    m, n, K = (int(x) for x in rng.integers(1, cap, 3))
    dens = float(rng.choice([0.05, 0.2, 0.5]))
    kind = rng.choice(["spmm", "spmv", "spmm_add", "spmm_bt", "sddmm", "mttkrp", "spgemm", "add", "mul"])
    if kind in ("spmm", "spmm_add", "spmm_bt", "spmv"):
        A = random_tensor(rng, (m, n), str(rng.choice(SPARSE)), dens, "A", device="cuda")
        if kind == "spmv":
            x = _dense(rng, (n,), "x")
            return f"y({i}) = A({i},{j}) * x({j})", {"A": A, "x": x}
        if kind == "spmm_bt":
            BT = _dense(rng, (K, n), "BT")
            fac = [f"A({i},{j})", f"BT({k},{j})"]
            rng.shuffle(fac)
            return f"C({i},{k}) = {fac[0]} * {fac[1]}", {"A": A, "BT": BT}
        B = _dense(rng, (n, K), "B")
        fac = [f"A({i},{j})", f"B({j},{k})"]
        rng.shuffle(fac)
        src = f"C({i},{k}) = {fac[0]} * {fac[1]}"
        if kind == "spmm_add":
            return src + f" + D({i},{k})", {"A": A, "B": B, "D": _dense(rng, (m, K), "D")}
        return src, {"A": A, "B": B}
    if kind == "sddmm":
        d = int(rng.integers(1, 300))
        M = random_tensor(rng, (m, n), "csr", dens, "M", device="cuda")
        fac = [f"M({i},{j})", f"Q({i},{k})", f"K({j},{k})"]
        rng.shuffle(fac)
        return f"S({i},{j}) = {' * '.join(fac)}", {"M": M, "Q": _dense(rng, (m, d), "Q"),
                                                   "K": _dense(rng, (n, d), "K")}
    if kind == "mttkrp":
        p, q, R = (int(x) for x in rng.integers(1, 12, 3))
        size = m * p * q
        flat = np.sort(rng.choice(size, size=max(1, int(size * dens)), replace=False))
        coords = np.stack(np.unravel_index(flat, (m, p, q)), axis=1)
        vals = rng.uniform(0, 1, len(coords)).astype(np.float32)
        T = st.coo_from_sorted_arrays(tuple(coords.T), vals, (m, p, q), name="T")
        r = names[3]
        # any output mode (CP-ALS runs all three)
        idx, ext = [i, j, k], [m, p, q]
        o = int(rng.integers(0, 3))
        (u, eu), (w, ew) = [(idx[t], ext[t]) for t in range(3) if t != o]
        return (f"M({idx[o]},{r}) = T({i},{j},{k}) * B({u},{r}) * C({w},{r})",
                {"T": T, "B": _dense(rng, (eu, R), "B"), "C": _dense(rng, (ew, R), "C")})
    if kind == "spgemm":
        A = random_tensor(rng, (m, n), "csr", dens, "A", device="cuda")
        B = random_tensor(rng, (n, K), "csr", dens, "B", device="cuda")
        return f"C({i},{k}) = A({i},{j}) * B({j},{k})", {"A": A, "B": B}
    A = random_tensor(rng, (m, n), "csr", dens, "A", device="cuda")
    B = random_tensor(rng, (m, n), "csr", float(rng.choice([0.05, 0.2, 0.5])), "B", device="cuda")
    op = "+" if kind == "add" else "*"
    return f"C({i},{j}) = A({i},{j}) {op} B({i},{j})", {"A": A, "B": B}


@pytest.mark.parametrize("block", range(8))
def test_hot_path_expressions_match_dense_evaluation(block):
    for seed in range(block * 50, (block + 1) * 50):
        rng = np.random.default_rng(7000 + seed)
        src, tensors = _hot_path_case(rng)
        e = st.parse(src, tensors)
        out, _, report = st.run_with_report(e)
        assert report["path"] == "sparse" and report["variants"], (seed, src)
        assert not any(v.startswith("generic") for v in report["variants"]), (seed, src, report["variants"])
        assert out.format == st.infer_format(e), (seed, src, out.format, st.infer_format(e))
        want = st.eval_dense(e)
        ok, worst = parity_gate(np.asarray(st.to_dense(out), dtype=np.float64), want, abs_bound(e, tensors), 1e-5)
        assert ok, f"seed {7000 + seed}: {src} worst {worst}"


def test_random_expressions_all_run_on_the_device():
    """The reference's random strategy: every expression runs (dedicated kernel or the
    device loop-nest walker) and matches the dense evaluation."""
    ran = 0
    for seed in range(120):
        rng = np.random.default_rng(1000 + seed)
        e = random_expression(rng, extent_cap=9, device="cuda")
        tensors = {a.tensor.name: a.tensor for a in e.accesses}
        out, _, _ = st.run_with_report(e)
        assert out.storage.values.is_cuda
        ran += 1
        want = st.eval_dense(e)
        ok, worst = parity_gate(np.asarray(st.to_dense(out), dtype=np.float64).reshape(want.shape), want,
                                abs_bound(e, tensors), 1e-5)
        assert ok, f"seed {1000 + seed}: {e} worst {worst}"
    assert ran > 0
