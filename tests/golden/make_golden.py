"""Generate golden fixtures by running the REAL reference engine.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every case draws seeded float32-rounded inputs, builds the reference tensors
with ``sparsetc.build_from_entries``/``from_dense``, runs ``sparsetc.run_with_report``
(schedule + tile 64 + execute, exactly the library entry, engine.py:667-717)
and stores inputs, the output's storage (level pos/crd + values), the
inferred/out format, loop order and op counters in ``tests/golden/<case>.npz``.
Nothing here is shipped; the GPU box only reads the .npz files.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import sparsetc as st  # noqa: E402
from sparsetc.tensor import CompressedLevel, CoordinateLevel  # noqa: E402


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def rand_sparse_entries(rng, shape, density, explicit_zero_frac=0.0, empty_rows=()):
    size = int(np.prod(shape))
    count = max(1, round(size * density))
    flat = rng.choice(size, size=count, replace=False)
    coords = np.stack(np.unravel_index(flat, shape), axis=1)
    if empty_rows:
        coords = coords[~np.isin(coords[:, 0], empty_rows)]
    vals = f32(rng.uniform(-1, 1, len(coords)))
    if explicit_zero_frac:
        vals[rng.random(len(vals)) < explicit_zero_frac] = 0.0
    return [(tuple(int(c) for c in co), float(v)) for co, v in zip(coords, vals)]


def storage_arrays(t, prefix):
    out = {}
    for k, lv in enumerate(t.storage.levels):
        if isinstance(lv, CompressedLevel):
            out[f"{prefix}_l{k}_pos"] = np.asarray(lv.pos)
            out[f"{prefix}_l{k}_crd"] = np.asarray(lv.crd)
        elif isinstance(lv, CoordinateLevel):
            out[f"{prefix}_l{k}_crd"] = np.asarray(lv.crd)
    out[f"{prefix}_vals"] = np.asarray(t.storage.values)
    out[f"{prefix}_shape"] = np.asarray(t.shape)
    out[f"{prefix}_modes"] = np.asarray(t.format.mode_ordering)
    out[f"{prefix}_levels"] = np.asarray([lv.value for lv in t.format.levels])
    return out


CASES = {}


def case(fn):
    CASES[fn.__name__] = fn
    return fn


def run_case(name, src, tensors, tile_size=64, tiling=True):
    e = st.parse(src, tensors)
    result, counter, report = st.run_with_report(e, tile_size=tile_size, tiling=tiling)
    arrays = {}
    for tname, t in tensors.items():
        arrays.update(storage_arrays(t, f"in_{tname}"))
    arrays.update(storage_arrays(result, "out"))
    arrays["out_dense"] = st.to_dense(result)
    meta = {
        "src": src,
        "inputs": list(tensors),
        "out_format": result.format.name(),
        "path": report["path"],
        "counters": None if counter is None else counter.as_dict(),
        "loop_order": None if report["schedule"] is None else report["schedule"]["loop_order"],
        "tiles": None if report["schedule"] is None else report["schedule"]["tiles"],
        "workspace": None if report["schedule"] is None else report["schedule"]["workspace"],
        "tiling": tiling,
        "tile_size": tile_size,
    }
    arrays["meta"] = np.asarray(json.dumps(meta))
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    return meta


@case
def spmm_csr_k13():
    rng = np.random.default_rng(101)
    A = st.build_from_entries((37, 29), st.csr(37, 29), rand_sparse_entries(rng, (37, 29), 0.2, 0.05, (3, 17)), "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (29, 13))), name="B")
    return run_case("spmm_csr_k13", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def spmm_csr_k130():
    rng = np.random.default_rng(102)
    A = st.build_from_entries((41, 33), st.csr(41, 33), rand_sparse_entries(rng, (41, 33), 0.15), "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (33, 130))), name="B")
    return run_case("spmm_csr_k130", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def spmm_csr_skewed():
    # power-law-ish rows: one very long row, many short, some empty
    rng = np.random.default_rng(103)
    n = 60
    entries = []
    for i in range(n):
        L = 55 if i == 7 else (0 if i % 9 == 4 else int(rng.integers(1, 4)))
        cols = np.sort(rng.choice(n, size=L, replace=False))
        entries += [((i, int(c)), float(f32(rng.uniform(-1, 1)))) for c in cols]
    A = st.build_from_entries((n, n), st.csr(n, n), entries, "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (n, 64))), name="B")
    return run_case("spmm_csr_skewed", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def spmm_csr_addend():
    rng = np.random.default_rng(104)
    A = st.build_from_entries((19, 23), st.csr(19, 23), rand_sparse_entries(rng, (19, 23), 0.25), "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (23, 8))), name="B")
    D = st.from_dense(f32(rng.uniform(-1, 1, (19, 8))), name="D")
    return run_case("spmm_csr_addend", "C(i,k) = A(i,j) * B(j,k) + D(i,k)", {"A": A, "B": B, "D": D})


@case
def spmv_csr():
    rng = np.random.default_rng(105)
    A = st.build_from_entries((31, 27), st.csr(31, 27), rand_sparse_entries(rng, (31, 27), 0.2), "A")
    x = st.from_dense(f32(rng.uniform(-1, 1, 27)), name="x")
    return run_case("spmv_csr", "y(i) = A(i,j) * x(j)", {"A": A, "x": x})


@case
def spmm_coo():
    rng = np.random.default_rng(106)
    A = st.build_from_entries((29, 21), st.coo(29, 21), rand_sparse_entries(rng, (29, 21), 0.12, 0.05), "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (21, 12))), name="B")
    return run_case("spmm_coo", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def spmm_dcsr():
    rng = np.random.default_rng(107)
    A = st.build_from_entries((26, 18), st.dcsr(26, 18), rand_sparse_entries(rng, (26, 18), 0.1), "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (18, 8))), name="B")
    return run_case("spmm_dcsr", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def spmm_csc():
    rng = np.random.default_rng(108)
    A = st.build_from_entries((22, 17), st.csc(22, 17), rand_sparse_entries(rng, (22, 17), 0.2), "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (17, 8))), name="B")
    return run_case("spmm_csc", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def sddmm_d5():
    rng = np.random.default_rng(109)
    M = st.build_from_entries((23, 31), st.csr(23, 31), rand_sparse_entries(rng, (23, 31), 0.2, 0.0, (5,)), "M")
    Q = st.from_dense(f32(rng.uniform(-1, 1, (23, 5))), name="Q")
    K = st.from_dense(f32(rng.uniform(-1, 1, (31, 5))), name="K")
    return run_case("sddmm_d5", "S(i,j) = M(i,j) * Q(i,d) * K(j,d)", {"M": M, "Q": Q, "K": K})


@case
def sddmm_d64():
    rng = np.random.default_rng(110)
    M = st.build_from_entries((17, 19), st.csr(17, 19), rand_sparse_entries(rng, (17, 19), 0.3), "M")
    Q = st.from_dense(f32(rng.standard_normal((17, 64))), name="Q")
    KT = st.from_dense(f32(rng.standard_normal((64, 19))), name="KT")
    return run_case("sddmm_d64", "S(i,j) = M(i,j) * Q(i,d) * KT(d,j)", {"M": M, "Q": Q, "KT": KT})


@case
def sddmm_d100():
    rng = np.random.default_rng(111)
    M = st.build_from_entries((9, 11), st.csr(9, 11), rand_sparse_entries(rng, (9, 11), 0.3), "M")
    Q = st.from_dense(f32(rng.standard_normal((9, 100))), name="Q")
    K = st.from_dense(f32(rng.standard_normal((11, 100))), name="K")
    return run_case("sddmm_d100", "S(i,j) = M(i,j) * Q(i,d) * K(j,d)", {"M": M, "Q": Q, "K": K})


@case
def sddmm_d300():
    # reduction wider than one 128-lane kernel block: three blocks summed, then the mask value
    rng = np.random.default_rng(115)
    M = st.build_from_entries((9, 12), st.csr(9, 12), rand_sparse_entries(rng, (9, 12), 0.3), "M")
    Q = st.from_dense(f32(rng.standard_normal((9, 300))), name="Q")
    K = st.from_dense(f32(rng.standard_normal((12, 300))), name="K")
    return run_case("sddmm_d300", "S(i,j) = M(i,j) * Q(i,d) * K(j,d)", {"M": M, "Q": Q, "K": K})


@case
def sddmm_multihead():
    rng = np.random.default_rng(112)
    M = st.build_from_entries((10, 10), st.csr(10, 10), rand_sparse_entries(rng, (10, 10), 0.3), "M")
    Q = st.from_dense(f32(rng.standard_normal((2, 10, 8))), name="Q")
    K = st.from_dense(f32(rng.standard_normal((2, 10, 8))), name="K")
    return run_case("sddmm_multihead", "Sc(h,i,j) = M(i,j) * Q(h,i,d) * K(h,j,d)", {"M": M, "Q": Q, "K": K})


@case
def pv_multihead():
    rng = np.random.default_rng(113)
    fmt = st.TensorFormat((2, 10, 10), (0, 1, 2),
                          (st.LevelFormat.DENSE, st.LevelFormat.DENSE, st.LevelFormat.COMPRESSED))
    ents = rand_sparse_entries(rng, (10, 10), 0.3)
    P_entries = [((h, i, j), float(f32(rng.uniform(0, 1)))) for h in range(2) for (i, j), _ in ents]
    P = st.build_from_entries((2, 10, 10), fmt, P_entries, "P")
    V = st.from_dense(f32(rng.standard_normal((2, 10, 8))), name="V")
    return run_case("pv_multihead", "O(h,i,d) = P(h,i,j) * V(h,j,d)", {"P": P, "V": V})


@case
def mttkrp_coo3():
    rng = np.random.default_rng(114)
    shape = (12, 10, 9)
    size = int(np.prod(shape))
    flat = np.sort(rng.choice(size, size=90, replace=False))
    coords = np.stack(np.unravel_index(flat, shape), axis=1)
    vals = f32(rng.uniform(0, 1, len(coords)))
    T = st.build_from_entries(shape, st.coo(*shape), [(tuple(map(int, c)), float(v)) for c, v in zip(coords, vals)], "T")
    B = st.from_dense(f32(rng.uniform(0, 1, (10, 6))), name="B")
    C = st.from_dense(f32(rng.uniform(0, 1, (9, 6))), name="C")
    return run_case("mttkrp_coo3", "M(i,r) = T(i,j,k) * B(j,r) * C(k,r)", {"T": T, "B": B, "C": C})


def _mttkrp_tensor(rng, shape, n):
    size = int(np.prod(shape))
    flat = np.sort(rng.choice(size, size=n, replace=False))
    coords = np.stack(np.unravel_index(flat, shape), axis=1)
    vals = f32(rng.uniform(0, 1, len(coords)))
    return st.build_from_entries(shape, st.coo(*shape), [(tuple(map(int, c)), float(v)) for c, v in zip(coords, vals)],
                                 "T")


@case
def mttkrp_mode2():
    # CP-ALS runs MTTKRP in every mode; the reference walks T in storage order for each
    rng = np.random.default_rng(140)
    T = _mttkrp_tensor(rng, (12, 10, 9), 110)
    A = st.from_dense(f32(rng.uniform(0, 1, (12, 5))), name="A")
    C = st.from_dense(f32(rng.uniform(0, 1, (9, 5))), name="C")
    return run_case("mttkrp_mode2", "M(j,r) = T(i,j,k) * A(i,r) * C(k,r)", {"T": T, "A": A, "C": C})


@case
def mttkrp_mode3():
    rng = np.random.default_rng(141)
    T = _mttkrp_tensor(rng, (8, 11, 13), 120)
    A = st.from_dense(f32(rng.uniform(0, 1, (8, 7))), name="A")
    B = st.from_dense(f32(rng.uniform(0, 1, (11, 7))), name="B")
    return run_case("mttkrp_mode3", "M(k,r) = T(i,j,k) * A(i,r) * B(j,r)", {"T": T, "A": A, "B": B})


@case
def kat_sddmm_worked():
    # reference tests/test_engine.py:12-19: D[0,1] == 44.0 with 3 mults
    A = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 1), 2.0)], name="A")
    B = st.from_dense([[1.0, 2.0], [3.0, 4.0]], name="B")
    C = st.from_dense([[5.0, 6.0], [7.0, 8.0]], name="C")
    return run_case("kat_sddmm_worked", "D(i,j) = A(i,j) * B(i,k) * C(k,j)", {"A": A, "B": B, "C": C},
                    tiling=False)


@case
def kat_spmv_worked():
    # reference tests/test_engine.py:22-28: y == [3, 8]
    A = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 0), 1.0), ((1, 1), 2.0)], name="A")
    x = st.from_dense([3.0, 4.0], name="x")
    return run_case("kat_spmv_worked", "y(i) = A(i,j) * x(j)", {"A": A, "x": x}, tiling=False)


@case
def kat_zero_kept():
    # arithmetic zeros are stored values (tests/test_engine.py:186-192), here via SDDMM
    M = st.build_from_entries((2, 3), st.csr(2, 3), [((0, 0), 1.0), ((1, 2), 0.0)], name="M")
    Q = st.from_dense([[1.0, 0.0], [2.0, 3.0]], name="Q")
    K = st.from_dense([[0.0, 5.0], [1.0, 1.0], [4.0, -1.0]], name="K")
    return run_case("kat_zero_kept", "S(i,j) = M(i,j) * Q(i,d) * K(j,d)", {"M": M, "Q": Q, "K": K})


@case
def counters_sddmm_fused():
    # tests/test_acceptance.py:119-131: nnz=100, K=16 -> 1700 mults
    rng = np.random.default_rng(7)
    flat = rng.choice(100 * 100, size=100, replace=False)
    vals = rng.uniform(-1.0, 1.0, size=100)
    entries = [((int(f) // 100, int(f) % 100), float(f32(v))) for f, v in zip(flat, vals)]
    A = st.build_from_entries((100, 100), st.csr(100, 100), entries, name="A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (100, 16))), name="B")
    C = st.from_dense(f32(rng.uniform(-1, 1, (16, 100))), name="C")
    return run_case("counters_sddmm_fused", "D(i,j) = A(i,j) * B(i,k) * C(k,j)", {"A": A, "B": B, "C": C})


@case
def spmm_csr_k130_untiled():
    rng = np.random.default_rng(102)
    A = st.build_from_entries((41, 33), st.csr(41, 33), rand_sparse_entries(rng, (41, 33), 0.15), "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (33, 130))), name="B")
    return run_case("spmm_csr_k130_untiled", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B}, tiling=False)


@case
def spmm_coo_k70():
    rng = np.random.default_rng(115)
    A = st.build_from_entries((25, 19), st.coo(25, 19), rand_sparse_entries(rng, (25, 19), 0.1), "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (19, 70))), name="B")
    return run_case("spmm_coo_k70", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def spmm_coo_untiled():
    rng = np.random.default_rng(106)
    A = st.build_from_entries((29, 21), st.coo(29, 21), rand_sparse_entries(rng, (29, 21), 0.12, 0.05), "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (21, 12))), name="B")
    return run_case("spmm_coo_untiled", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B}, tiling=False)


@case
def sddmm_d100_untiled():
    rng = np.random.default_rng(111)
    M = st.build_from_entries((9, 11), st.csr(9, 11), rand_sparse_entries(rng, (9, 11), 0.3), "M")
    Q = st.from_dense(f32(rng.standard_normal((9, 100))), name="Q")
    K = st.from_dense(f32(rng.standard_normal((11, 100))), name="K")
    return run_case("sddmm_d100_untiled", "S(i,j) = M(i,j) * Q(i,d) * K(j,d)", {"M": M, "Q": Q, "K": K},
                    tiling=False)


@case
def mttkrp_coo3_r70():
    rng = np.random.default_rng(116)
    shape = (8, 7, 6)
    size = int(np.prod(shape))
    flat = np.sort(rng.choice(size, size=40, replace=False))
    coords = np.stack(np.unravel_index(flat, shape), axis=1)
    vals = f32(rng.uniform(0, 1, len(coords)))
    T = st.build_from_entries(shape, st.coo(*shape), [(tuple(map(int, c)), float(v)) for c, v in zip(coords, vals)], "T")
    B = st.from_dense(f32(rng.uniform(0, 1, (7, 70))), name="B")
    C = st.from_dense(f32(rng.uniform(0, 1, (6, 70))), name="C")
    return run_case("mttkrp_coo3_r70", "M(i,r) = T(i,j,k) * B(j,r) * C(k,r)", {"T": T, "B": B, "C": C})


@case
def spmm_csr_ki_out():
    # output spelled C(k,i): the reference picks order [k,i,j] with no tiles
    rng = np.random.default_rng(117)
    A = st.build_from_entries((15, 13), st.csr(15, 13), rand_sparse_entries(rng, (15, 13), 0.25), "A")
    B = st.from_dense(f32(rng.uniform(-1, 1, (13, 6))), name="B")
    return run_case("spmm_csr_ki_out", "C(k,i) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def spmm_csr_bt():
    # dense operand read transposed: BT(k,j)
    rng = np.random.default_rng(118)
    A = st.build_from_entries((14, 12), st.csr(14, 12), rand_sparse_entries(rng, (14, 12), 0.25), "A")
    BT = st.from_dense(f32(rng.uniform(-1, 1, (9, 12))), name="BT")
    return run_case("spmm_csr_bt", "C(i,k) = A(i,j) * BT(k,j)", {"A": A, "BT": BT})


@case
def dense_matmul():
    # all-dense dispatch (tests/test_acceptance.py:209-225)
    A = st.from_dense([[1.0, 2.0], [3.0, 4.0]], name="A")
    B = st.from_dense([[5.0, 6.0], [7.0, 8.0]], name="B")
    return run_case("dense_matmul", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def spgemm_csr():
    # sparse x sparse: CSR out, workspace over k, empty rows on both sides
    rng = np.random.default_rng(119)
    A = st.build_from_entries((23, 17), st.csr(23, 17), rand_sparse_entries(rng, (23, 17), 0.2, 0.05, (2, 11)), "A")
    B = st.build_from_entries((17, 19), st.csr(17, 19), rand_sparse_entries(rng, (17, 19), 0.25, 0.0, (4,)), "B")
    return run_case("spgemm_csr", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def spgemm_csr_skewed():
    # one dense row of A and one dense row of B: long product runs per output coordinate
    rng = np.random.default_rng(120)
    n = 40
    ents_a = rand_sparse_entries(rng, (n, n), 0.05)
    ents_a = [e for e in ents_a if e[0][0] != 5] + [((5, j), float(f32(rng.uniform(-1, 1)))) for j in range(n)]
    ents_b = rand_sparse_entries(rng, (n, n), 0.08)
    ents_b = [e for e in ents_b if e[0][0] != 9] + [((9, k), float(f32(rng.uniform(-1, 1)))) for k in range(n)]
    A = st.build_from_entries((n, n), st.csr(n, n), ents_a, "A")
    B = st.build_from_entries((n, n), st.csr(n, n), ents_b, "B")
    return run_case("spgemm_csr_skewed", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def kat_spgemm_zero_kept():
    # products that cancel still store their coordinate (tests/test_engine.py:186-192 semantics)
    A = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 0), 1.0), ((0, 1), 1.0), ((1, 1), 2.0)], name="A")
    B = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 0), 3.0), ((1, 0), -3.0), ((1, 1), 0.5)], name="B")
    return run_case("kat_spgemm_zero_kept", "C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})


@case
def ewise_add_csr():
    rng = np.random.default_rng(121)
    A = st.build_from_entries((21, 26), st.csr(21, 26), rand_sparse_entries(rng, (21, 26), 0.2, 0.05, (3,)), "A")
    B = st.build_from_entries((21, 26), st.csr(21, 26), rand_sparse_entries(rng, (21, 26), 0.3, 0.0, (3, 8)), "B")
    return run_case("ewise_add_csr", "C(i,j) = A(i,j) + B(i,j)", {"A": A, "B": B})


@case
def ewise_mul_csr():
    rng = np.random.default_rng(122)
    A = st.build_from_entries((21, 26), st.csr(21, 26), rand_sparse_entries(rng, (21, 26), 0.35, 0.05, (6,)), "A")
    B = st.build_from_entries((21, 26), st.csr(21, 26), rand_sparse_entries(rng, (21, 26), 0.3, 0.0, (8,)), "B")
    return run_case("ewise_mul_csr", "C(i,j) = A(i,j) * B(i,j)", {"A": A, "B": B})


@case
def spmv_coo():
    # SpMV with a COO matrix: compressed-vector output over the rows holding entries
    rng = np.random.default_rng(123)
    A = st.build_from_entries((27, 19), st.coo(27, 19), rand_sparse_entries(rng, (27, 19), 0.1, 0.05), "A")
    x = st.from_dense(f32(rng.uniform(-1, 1, 19)), name="x")
    return run_case("spmv_coo", "y(i) = A(i,j) * x(j)", {"A": A, "x": x})


@case
def spmv_csc():
    rng = np.random.default_rng(124)
    A = st.build_from_entries((21, 16), st.csc(21, 16), rand_sparse_entries(rng, (21, 16), 0.15), "A")
    x = st.from_dense(f32(rng.uniform(-1, 1, 16)), name="x")
    return run_case("spmv_csc", "y(i) = A(i,j) * x(j)", {"A": A, "x": x})


def main():
    only = set(sys.argv[1:])
    index = {}
    idx_path = OUT / "index.json"
    if only and idx_path.exists():
        index = json.loads(idx_path.read_text())
    for name, fn in CASES.items():
        if only and name not in only:
            continue
        index[name] = fn()
        print(f"{name}: {index[name]['out_format']} counters={index[name]['counters']}")
    (OUT / "index.json").write_text(json.dumps(index, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
