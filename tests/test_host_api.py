"""Host-side API parity with the reference: formats, parser, format inference,
planner and tiler goldens, and storage construction. The expectations restate
the reference's own tests (cited per test); no GPU needed — tensors are built
on the default device (CPU here, CUDA on the GPU box).
"""

import json

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as hs

import paper_2405_16883_b200 as st
from paper_2405_16883_b200.expr import Add, Mul, ParseError
from paper_2405_16883_b200.format_inference import LevelClass, infer_level
from paper_2405_16883_b200.scheduler import CostModel, IterationKind, move_cost
from paper_2405_16883_b200.tiling import expanded_loops

from helpers import MATRIX_FORMATS, random_expression, random_tensor


def names(vs):
    return [v.name for v in vs]


def zeros(**shapes):
    return {n: st.from_dense(np.zeros(s), name=n) for n, s in shapes.items()}


# ---- formats (tests/test_formats.py) -------------------------------------------------

def test_named_formats():
    assert st.csr(3, 4).levels == (st.LevelFormat.DENSE, st.LevelFormat.COMPRESSED)
    assert st.csc(3, 4).mode_ordering == (1, 0)
    assert st.dcsr(3, 4).levels == (st.LevelFormat.COMPRESSED,) * 2
    assert st.coo(3, 4).levels == (st.LevelFormat.COORDINATE,) * 2
    for n in MATRIX_FORMATS:
        assert st.format_by_name(n, (3, 4)).name() == n
    assert st.csc(3, 4).level_extent(0) == 4
    assert st.level_is_sparse(st.csc(2, 2), 0) and not st.level_is_sparse(st.csc(2, 2), 1)
    g = st.csr(3, 4).with_mode_ordering((1, 0))
    assert g.levels == (st.LevelFormat.COMPRESSED, st.LevelFormat.DENSE)


def test_bad_formats():
    L = st.LevelFormat
    for args in [((2, 2), (0, 1), (L.COORDINATE, L.DENSE)), ((2, 2), (0, 0), (L.DENSE, L.DENSE)),
                 ((2,), (0, 1), (L.DENSE, L.DENSE)), ((0, 2), (0, 1), (L.DENSE, L.DENSE))]:
        with pytest.raises(ValueError):
            st.TensorFormat(*args)
    with pytest.raises(ValueError):
        st.format_by_name("ellpack", (2, 2))


# ---- parser (tests/test_expr.py) ------------------------------------------------------

def test_parse_and_variables():
    b = zeros(A=(4, 5), B=(4, 3), C=(3, 5))
    e = st.parse("D(i,j) = A(i,j) * B(i,k) * C(k,j)", b)
    assert names(e.output_indices) == ["i", "j"]
    assert names(st.get_index_variables(e)) == ["i", "j", "k"]
    assert {v.name for v in st.get_reduction_variables(e)} == {"k"}
    b = zeros(A=(2, 2), B=(2, 2), C=(2, 2))
    e = st.parse("C(i,k) = A(i,j) * B(j,k)", b)
    assert names(st.get_index_variables(e)) == ["i", "k", "j"]
    e = st.parse("D(i,j) = A(i,k) * B(k,j) + C(i,j)", b)
    assert isinstance(e.rhs, Add) and isinstance(e.rhs.lhs, Mul)
    assert [a.name for a in e.terms()[0]] == ["A", "B"]
    assert st.render(e) == "D(i,j) = A(i,k) * B(k,j) + C(i,j)"
    assert st.parse(st.render(e), b) == e


def test_parse_errors():
    b = zeros(A=(2, 2))
    for src in ["C(i,j) = Z(i,j)", "C(i) = A(i)", "C(i,i) = A(i,i)", "C(i,m) = A(i,j)", "A(i,j)",
                "C(i,j) = A(i,j) *", "C(i,j) = A(i,j) A(i,j)", "C(i,j) = + A(i,j)"]:
        with pytest.raises(ParseError):
            st.parse(src, b)
    with pytest.raises(st.ShapeError):
        st.parse("C(i,k) = A(i,j) * B(j,k)", zeros(A=(2, 3), B=(4, 2)))


def test_einsum_desugar():
    b = zeros(A=(4, 5), B=(5, 6))
    e = st.parse_einsum("ij,jk->ik", [b["A"], b["B"]])
    assert st.render(e) == "Out(i,k) = A(i,j) * B(j,k)"
    with pytest.raises(ParseError):
        st.parse_einsum("ij,jk", [b["A"], b["B"]])
    with pytest.raises(ParseError):
        st.parse_einsum("ij->ij", [b["A"], b["B"]])


@given(seed=hs.integers(0, 2**31))
@settings(max_examples=30, deadline=None)
def test_render_parse_round_trip(seed):
    e = random_expression(np.random.default_rng(seed), extent_cap=4)
    bindings = {a.tensor.name: a.tensor for a in e.accesses}
    assert st.parse(st.render(e), bindings) == e


# ---- format inference (tests/test_format_inference.py, acceptance criterion 3) ------

def _abc(r):
    return {"A": random_tensor(r, (4, 3), "csr", 0.4, "A"),
            "B": random_tensor(r, (3, 5), "csr", 0.4, "B"),
            "C": random_tensor(r, (4, 5), "dcsr", 0.4, "C")}


def test_inference_goldens():
    e = st.parse("D(i,j) = A(i,k) * B(k,j) + C(i,j)", _abc(np.random.default_rng(0)))
    assert st.infer_format(e).name() == "csr"
    assert infer_level(e.rhs.lhs, st.IndexVar("i")) is LevelClass.DENSE
    assert infer_level(e.rhs.lhs, st.IndexVar("j")) is LevelClass.SPARSE
    tree = st.explain_format(e)
    assert tree["format"] == "csr" and tree["levels"][0]["derivation"]["op"] == "add"
    r = np.random.default_rng(2)
    A = random_tensor(r, (4, 3), "csr", 0.5, "A")
    Bd = st.from_dense(np.ones((3, 5)), name="Bd")
    assert st.infer_format(st.parse("C(i,k) = A(i,j) * Bd(j,k)", {"A": A, "Bd": Bd})).name() == "dense"
    Ac = random_tensor(r, (4, 3), "coo", 0.5, "Ac")
    f = st.infer_format(st.parse("C(i,k) = Ac(i,j) * Bd(j,k)", {"Ac": Ac, "Bd": Bd}))
    assert f.levels == (st.LevelFormat.COMPRESSED, st.LevelFormat.DENSE)


# ---- scheduler goldens (tests/test_scheduler.py, acceptance criteria 1-2) -----------

def spgemm(seed=0, n=6):
    r = np.random.default_rng(seed)
    return st.parse("C(i,k) = A(i,j) * B(j,k)", {"A": random_tensor(r, (n, n), "csr", 0.3, "A"),
                                                 "B": random_tensor(r, (n, n), "csr", 0.3, "B")})


def spmm(seed=0, n=6, k=4):
    r = np.random.default_rng(seed)
    A = random_tensor(r, (n, n), "csr", 0.3, "A")
    return st.parse("C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": st.from_dense(r.uniform(-1, 1, (n, k)), name="B")})


def test_sort_by_sparsity_goldens():
    e = spgemm()
    assert names(st.sort_by_sparsity(st.get_index_variables(e), e)) == ["j", "i", "k"]
    b = {n: st.from_dense(np.ones((4, 4)), name=n) for n in "AB"}
    e = st.parse("C(i,k) = A(i,j) * B(j,k)", b)
    assert names(st.sort_by_sparsity(st.get_index_variables(e), e)) == ["i", "j", "k"]
    r = np.random.default_rng(0)
    A = random_tensor(r, (5, 4), "csr", 0.4, "A")
    e = st.parse("y(i) = A(i,j) * x(j)", {"A": A, "x": st.from_dense(np.ones(4), name="x")})
    assert names(st.sort_by_sparsity(st.get_index_variables(e), e)) == ["j", "i"]


def test_gustavson_golden_and_moves():
    s = st.schedule(spgemm())
    assert names(s.loop_order) == ["i", "j", "k"] and s.transposes == ()
    ws = s.workspace
    assert ws.dimensions == 1 and names(ws.ws_indices) == ["k"]
    assert names(ws.producer_loops) == ["j", "k"] and ws.split_var.name == "j"
    first, second = s.moves[0], s.moves[1]
    assert first.accepted and dict(first.components) == {
        "filter_loss": 4.0, "workspace": -2.0, "transposes": -3.0, "dense_iteration": 0.0}
    assert first.cost == -1.0
    assert not second.accepted and second.cost == 1005.0
    kinds = {l.var.name: l.kind for l in s.loops}
    assert kinds == {"i": IterationKind.DENSE_COUNT, "j": IterationKind.SPARSE_INTERSECT,
                     "k": IterationKind.SPARSE_ITERATE}
    jl = next(l for l in s.loops if l.var.name == "j")
    assert set(jl.filters) == {"A", "B"} and jl.is_reduction
    d = json.loads(json.dumps(st.schedule_to_dict(s)))
    assert d["loop_order"] == ["i", "j", "k"] and d["workspace"]["dimensions"] == 1


def test_inner_product_never_emitted_and_weights():
    for seed in range(8):
        assert names(st.schedule(spgemm(seed)).loop_order) in (["i", "j", "k"], ["j", "i", "k"])
    s = st.schedule(spgemm(), weights=CostModel(w_filter_loss=100.0))
    assert not s.moves[0].accepted
    e = spgemm()
    out = st.infer_format(e)
    order = list(st.sort_by_sparsity(st.get_index_variables(e), e))
    assert move_cost(e, out, order, order[0], 1)[0] == -1.0
    with pytest.raises(ValueError):
        move_cost(e, out, order, order[0], 0)


def test_spmm_and_transpose_goldens():
    s = st.schedule(spmm())
    assert names(s.loop_order) == ["i", "j", "k"] and s.workspace is None and s.transposes == ()
    r = np.random.default_rng(0)
    A = random_tensor(r, (4, 4), "csr", 0.5, "A")
    B = random_tensor(r, (4, 4), "csc", 0.25, "B")
    s = st.schedule(st.parse("C(i,j) = A(i,j) * B(i,j)", {"A": A, "B": B}))
    assert names(s.loop_order) == ["i", "j"] and s.transposes == (("B", (0, 1)),)
    r = np.random.default_rng(0)
    A = random_tensor(r, (4, 5), "csc", 0.4, "A")
    s = st.schedule(st.parse("y(i) = A(i,j) * x(j)", {"A": A, "x": st.from_dense(np.ones(5), name="x")}))
    assert names(s.loop_order) == ["j", "i"] and s.transposes == ()


def test_scheduler_determinism_and_budget():
    a, b = st.schedule(spgemm(3)), st.schedule(spgemm(3))
    assert a.loop_order == b.loop_order and a.moves == b.moves
    assert len(st.schedule(spgemm()).moves) <= 9


# ---- tiling goldens (tests/test_tiling.py, acceptance criterion 4) ------------------

def test_tiling_goldens():
    r = np.random.default_rng(0)
    A = random_tensor(r, (8, 6), "csr", 0.3, "A")
    e = st.parse("C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": st.from_dense(r.uniform(-1, 1, (6, 5)), name="B")})
    assert {v.name for v in st.tile(e, st.schedule(e), 64).tiles} == {"k"}
    dense = {n: st.from_dense(np.ones((6, 6)), name=n) for n in "AB"}
    e = st.parse("C(i,k) = A(i,j) * B(j,k)", dense)
    s = st.tile(e, st.schedule(e), 4)
    assert {v.name for v in s.tiles} == {"i", "j", "k"}
    assert [(x.var.name, x.role) for x in expanded_loops(s)] == [
        ("i", "block"), ("k", "block"), ("i", "intra"), ("j", "block"), ("j", "intra"), ("k", "intra")]
    Bm = st.from_dense(r.uniform(-1, 1, (8, 4)), name="Bm")
    Cm = st.from_dense(r.uniform(-1, 1, (4, 6)), name="Cm")
    e = st.parse("D(i,j) = A(i,j) * Bm(i,k) * Cm(k,j)", {"A": A, "Bm": Bm, "Cm": Cm})
    assert {v.name for v in st.tile(e, st.schedule(e), 64).tiles} == {"k"}
    e = spgemm(2, 5)
    assert st.tile(e, st.schedule(e), 4).tiles == ()
    assert all(x.role == "full" for x in expanded_loops(st.schedule(e)))
    with pytest.raises(ValueError):
        st.tile(e, st.schedule(e), 0)


# ---- storage construction (tests/test_tensor.py) --------------------------------------

def test_storage_kats():
    t = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 0), 1.0), ((1, 1), 2.0)])
    assert t.storage.levels[1].pos.tolist() == [0, 1, 2]
    assert t.storage.levels[1].crd.tolist() == [0, 1]
    assert t.storage.values.tolist() == [1.0, 2.0]
    t = st.build_from_entries((2, 2), st.coo(2, 2), [((1, 0), 3.0), ((0, 1), 4.0)])
    assert t.storage.levels[0].crd.tolist() == [0, 1] and t.storage.levels[1].crd.tolist() == [1, 0]
    assert t.storage.values.tolist() == [4.0, 3.0]
    t = st.build_from_entries((3, 3), st.dcsr(3, 3), [])
    assert t.storage.levels[0].pos.tolist() == [0, 0] and st.nnz(t) == 0
    t = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 1), 1.5), ((0, 1), 2.0)])
    assert st.nnz(t) == 1 and st.to_dense(t)[0, 1] == 3.5
    t = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 1), 0.0)])
    assert st.nnz(t) == 1 and st.nnz(st.convert(t, st.coo(2, 2))) == 1
    t = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 1), 1.0), ((1, 0), 2.0)])
    c = st.convert(t, st.csc(2, 2))
    assert c.storage.levels[1].pos.tolist() == [0, 1, 2] and c.storage.levels[1].crd.tolist() == [1, 0]
    assert c.storage.values.tolist() == [2.0, 1.0]


def test_storage_errors():
    with pytest.raises(IndexError):
        st.build_from_entries((2, 2), st.csr(2, 2), [((2, 0), 1.0)])
    with pytest.raises(st.ShapeError):
        st.build_from_entries((2, 2), st.csr(2, 2), [((0,), 1.0)])
    with pytest.raises(st.ShapeError):
        st.build_from_entries((2, 3), st.csr(3, 2), [])
    with pytest.raises(st.ShapeError):
        st.convert(st.build_from_entries((2, 3), st.csr(2, 3), []), st.csr(3, 2))


def test_three_level_and_from_arrays():
    fmt = st.TensorFormat((2, 3, 2), (0, 1, 2), (st.LevelFormat.DENSE, st.LevelFormat.COMPRESSED,
                                                  st.LevelFormat.COMPRESSED))
    ents = [((0, 1, 0), 2.0), ((1, 2, 1), 3.0), ((0, 1, 1), 4.0)]
    t = st.build_from_entries((2, 3, 2), fmt, ents)
    dense = np.zeros((2, 3, 2))
    for c, v in ents:
        dense[c] = v
    assert np.array_equal(st.to_dense(t), dense)
    assert np.array_equal(st.to_dense(st.convert(t, st.coo(2, 3, 2))), dense)
    coords = np.array([c for c, _ in ents] + [((0, 1, 0))])
    vals = np.array([v for _, v in ents] + [1.0])
    u = st.from_arrays((2, 3, 2), fmt, coords, vals)
    dense[0, 1, 0] += 1.0
    assert np.array_equal(st.to_dense(u), dense)


@given(data=hs.data())
@settings(max_examples=40, deadline=None)
def test_round_trip_between_all_formats(data):
    r = np.random.default_rng(data.draw(hs.integers(0, 2**31)))
    t = random_tensor(r, (5, 4), str(r.choice(MATRIX_FORMATS)), 0.35, "T")
    target = st.format_by_name(str(r.choice(MATRIX_FORMATS)), (5, 4))
    assert np.array_equal(st.to_dense(st.convert(t, target)), st.to_dense(t))


@given(seed=hs.integers(0, 2**31), perm_seed=hs.integers(0, 2**31))
@settings(max_examples=30, deadline=None)
def test_build_is_order_insensitive(seed, perm_seed):
    r = np.random.default_rng(seed)
    ents = [((int(r.integers(0, 5)), int(r.integers(0, 4))), float(r.uniform(-1, 1))) for _ in range(12)]
    fmt = st.format_by_name(str(r.choice(MATRIX_FORMATS)), (5, 4))
    a = st.build_from_entries((5, 4), fmt, ents)
    sh = list(ents)
    np.random.default_rng(perm_seed).shuffle(sh)
    b = st.build_from_entries((5, 4), fmt, sh)
    assert np.array_equal(a.storage.values.cpu().numpy(), b.storage.values.cpu().numpy())
    for la, lb in zip(a.storage.levels, b.storage.levels):
        for attr in ("pos", "crd"):
            if hasattr(la, attr):
                assert np.array_equal(getattr(la, attr).cpu().numpy(), getattr(lb, attr).cpu().numpy())


def test_storage_matches_reference_goldens():
    """Input tensors built here have the reference's exact pos/crd (fixtures)."""
    from conftest import load_golden

    g = load_golden("spmm_coo")
    rows, cols, vals = g["in_A_l0_crd"], g["in_A_l1_crd"], g["in_A_vals"]
    ents = [((int(i), int(j)), float(v)) for i, j, v in zip(rows[::-1], cols[::-1], vals[::-1])]
    for fmt_name in ("csr", "dcsr", "csc", "coo"):
        t = st.build_from_entries((29, 21), st.format_by_name(fmt_name, (29, 21)), ents)
        d = st.to_dense(t)
        assert np.array_equal(d[rows, cols], vals)
        assert st.nnz(t) == len(vals)
    g = load_golden("spmm_csc")
    pos, crd = g["in_A_l1_pos"], g["in_A_l1_crd"]
    col_of = np.repeat(np.arange(len(pos) - 1), np.diff(pos))
    ents = [((int(i), int(j)), float(v)) for i, j, v in zip(crd, col_of, g["in_A_vals"])]
    t = st.build_from_entries((22, 17), st.csc(22, 17), ents)
    assert t.storage.levels[1].pos.tolist() == pos.tolist()
    assert t.storage.levels[1].crd.tolist() == crd.tolist()



def test_oracle_module_alias():
    """`from sparsetc.oracle import eval_dense` (reference __init__.py:27) has a counterpart."""
    from paper_2405_16883_b200.oracle import eval_dense

    assert eval_dense is st.eval_dense


def test_build_from_entries_scalar_and_exact_duplicate_sum():
    """Duplicates are summed exactly (fsum, reference tensor.py:238-241), scalars included."""
    t = st.build_from_entries((), st.dense_format(()), [((), 1.5), ((), 2.25)], device="cpu")
    assert float(st.to_dense(t)) == 3.75
    t = st.build_from_entries((2, 3), st.csr(2, 3), [((0, 1), 1e16), ((0, 1), 1.0), ((0, 1), -1e16), ((1, 2), 5.0)],
                              device="cpu")
    assert st.to_dense(t)[0, 1] == 1.0 and st.nnz(t) == 2


def test_storage_buffers_are_read_only_and_numpy_convertible():
    """Level and value buffers behave like the reference's frozen arrays (tensor.py:53-56,
    71-72): assignment raises ValueError, numpy sees a read-only copy; torch ops on them
    return ordinary tensors and the buffers alias the device memory (no copy)."""
    import torch

    from paper_2405_16883_b200.tensor import StorageArray

    t = st.from_dense(np.array([[1.0, 0, 2], [0, 3, 0]]), st.csr(2, 3), name="T", device="cpu")
    lv = t.storage.levels[1]
    for buf in (lv.pos, lv.crd, t.storage.values):
        assert type(buf) is StorageArray
        with pytest.raises(ValueError):
            buf[0] = 1
        a = np.asarray(buf)
        assert not a.flags.writeable and np.array_equal(a, buf.numpy())
    assert np.array_equal(np.diff(lv.pos), [2, 1]) and lv.pos[-1] == st.nnz(t)
    assert type(t.storage.values * 2) is torch.Tensor and type(t.storage.values[1:]) is torch.Tensor
    c = st.convert(t, st.coo(2, 3))
    assert type(c.storage.values) is StorageArray
    assert np.array_equal(st.to_dense(c), st.to_dense(t))
