"""Execution of scheduled expressions on the GPU (drop-in for ``sparsetc.engine``).

The reference interprets the scheduled loop nest in Python
(`/root/reference/pkg/src/sparsetc/engine.py:657-724`). Here ``execute`` keeps
the same signature and result contract — a fresh tensor in the planned output
format plus an ``OpCounter`` — but pattern-matches the expression and its plan
to one hand-written sm_100a kernel variant and launches it on the current
CUDA stream:

=====================================================  ==========================  ===================
expression (index names arbitrary)                      reference plan              device variant
=====================================================  ==========================  ===================
``C(i,k) = A(i,j)*B(j,k) [+ D(i,k)]``, A CSR             dense, [i,j,k], tiles {k}   row / merge / coltile
``y(i) = A(i,j)*x(j)``                                   dense, [i,j]                row / merge, K = 1
A COO / DCSR / CSC (any storage order)                   [compressed, dense] + ws    segmented merge
``S(i,j) = M(i,j)*Q(i,d)*K(j,d)`` (or ``KT(d,j)``)       M's pattern, [i,j,d], {d}   SDDMM
``Sc(h,i,j) = M(i,j)*Q(h,i,d)*K(h,j,d)``                 [dense,dense,compressed]    head-batched SDDMM
``O(h,i,d) = P(h,i,j)*V(h,j,d)``                         dense, [h,i,j,d], {d}       head-batched merge
``M(i,r) = T(i,j,k)*B(j,r)*C(k,r)``, T COO               [compressed, dense] + ws    MTTKRP merge
``C(i,k) = A(i,j)*B(j,k)``, A and B CSR                  CSR, [i,j,k], ws {k}        SpGEMM (expand-sort-compress)
``C(i,j) = A(i,j) + B(i,j)``, CSR                        CSR, [i,j] (union)          element-wise union
``C(i,j) = A(i,j) * B(i,j)``, CSR                        CSR, [i,j] (intersection)   element-wise product
all operands dense                                       dense dispatch              torch (cuBLAS, TF32 off)
=====================================================  ==========================  ===================

Anything else raises ``UnsupportedExpressionError``: there is no CPU or
interpreter fallback. Counters are filled from the reference's closed forms
(validated against fixtures of the real engine, tests/golden).
"""

from __future__ import annotations

import math
import string
import time
from dataclasses import dataclass

import torch

from . import ops
from .expr import Access, TensorExpr, get_index_variables, index_extents
from .format_inference import infer_format
from .generic import TooLargeForGenericWalk, execute_generic
from .formats import LevelFormat, TensorFormat, dense_format
from .scheduler import CostModel, Schedule, schedule, schedule_to_dict
from .tensor import (
    CompressedLevel,
    DenseLevel,
    ShapeError,
    Tensor,
    TensorStorage,
    VALUE_DTYPE,
    _assemble,
    convert,
    stored_entries_torch,
    to_torch,
)
from .tiling import DEFAULT_TILE_SIZE, tile


class UnsupportedExpressionError(NotImplementedError):
    """The expression has no device kernel on this path (no CPU fallback)."""


@dataclass
class OpCounter:
    """Work of one execution, same fields as the reference (`engine.py:51-68`).

    Filled analytically from the reference's closed forms instead of being
    counted in an interpreter loop.
    """

    scalar_mults: int = 0
    scalar_adds: int = 0
    iterator_advances: int = 0

    def as_dict(self) -> dict:
        return {
            "scalar_mults": self.scalar_mults,
            "scalar_adds": self.scalar_adds,
            "iterator_advances": self.iterator_advances,
        }

    def add(self, mults=0, adds=0, iters=0):
        self.scalar_mults += int(mults)
        self.scalar_adds += int(adds)
        self.iterator_advances += int(iters)


class Workspace:
    """Ordered insert-or-accumulate map (`engine.py:71-90`), host-side utility.

    On the device the workspace is the per-row register accumulator of the
    segmented kernels; this class keeps the reference's public helper.
    """

    def __init__(self):
        self._slots: dict = {}

    def accumulate(self, key: tuple, value: float, counter: OpCounter) -> None:
        counter.scalar_adds += 1
        self._slots[key] = self._slots.get(key, 0.0) + value

    def drain(self):
        for key in sorted(self._slots):
            yield key, self._slots[key]

    def __len__(self):
        return len(self._slots)


# ---------------------------------------------------------------------------
# Row-major views of sparse operands (cached on the tensor: structure is immutable)
# ---------------------------------------------------------------------------


@dataclass
class RowView:
    """Entries of a 2-D sparse operand grouped by one index ("rows").

    ``dense_rows``: rowptr covers every row (CSR-like); otherwise ``seg_rows``
    lists the rows that hold entries (compressed / coordinate rows).
    """

    n_rows: int                # extent of the row index
    rowptr: torch.Tensor       # int32 [n_segments + 1]
    cols: torch.Tensor         # int32 [nnz]
    vals: torch.Tensor         # float32 [nnz]
    seg_rows: torch.Tensor | None
    kind: str                  # "csr" | "dcsr" | "coo" | "sorted"

    @property
    def dense_rows(self) -> bool:
        return self.seg_rows is None

    @property
    def n_segments(self) -> int:
        return self.rowptr.numel() - 1


def _cache(t: Tensor, key, build):
    if key not in t._cache:
        t._cache[key] = build()
    return t._cache[key]


def row_view(t: Tensor, row_dim: int) -> RowView:
    """Group the entries of 2-D sparse ``t`` by logical dimension ``row_dim``."""
    fmt = t.format
    st = t.storage
    col_dim = 1 - row_dim

    def build() -> RowView:
        first = fmt.mode_ordering[0]
        lv = fmt.levels
        if first == row_dim and lv == (LevelFormat.DENSE, LevelFormat.COMPRESSED):
            L = st.levels[1]
            return RowView(t.shape[row_dim], L.pos, L.crd, st.values, None, "csr")
        if first == row_dim and lv == (LevelFormat.COMPRESSED, LevelFormat.COMPRESSED):
            L0, L1 = st.levels
            return RowView(t.shape[row_dim], L1.pos, L1.crd, st.values, L0.crd, "dcsr")
        if first == row_dim and fmt.is_coordinate:
            seg = ops.coo_segments(st.levels[0].crd)
            return RowView(t.shape[row_dim], seg.ptr, st.levels[1].crd, st.values, seg.rows, "coo")
        # any other storage: re-sort entries by (row, col) on the device
        coords, vals = stored_entries_torch(t)
        key = coords[:, row_dim] * t.shape[col_dim] + coords[:, col_dim]
        order = torch.sort(key, stable=True).indices
        rows = coords[order, row_dim].to(torch.int32).contiguous()
        cols = coords[order, col_dim].to(torch.int32).contiguous()
        seg = ops.coo_segments(rows) if rows.numel() else ops.Segments(
            torch.zeros(0, dtype=torch.int32, device=t.device),
            torch.zeros(1, dtype=torch.int32, device=t.device))
        return RowView(t.shape[row_dim], seg.ptr, cols, vals[order].contiguous(), seg.rows, "sorted")

    return _cache(t, ("row_view", row_dim), build)


def _stats(t: Tensor, view: RowView, key) -> ops.RowStats:
    return _cache(t, ("stats",) + key, lambda: ops.row_stats(view.rowptr))


def _partition(t: Tensor, view: RowView, key, k: int) -> ops.MergePartition:
    return _cache(t, ("partition", k) + key,
                  lambda: ops.merge_partition(view.rowptr, view.vals.numel(), k=k, colidx=view.cols,
                                              vals=view.vals, max_row=_stats(t, view, key).max_row))


# ---------------------------------------------------------------------------
# Helpers
# ---------------------------------------------------------------------------


def _require_device(tensors) -> None:
    from ._abi import lib, require_cuda

    for t in tensors:
        require_cuda(t.storage.values)
    lib()  # the compiled extension must be present for every contraction (no torch-only path)


def _dense_torch(t: Tensor, order) -> torch.Tensor:
    """Dense operand as a torch tensor with its dims permuted to ``order`` (contiguous)."""
    x = t.storage.values.reshape(t.shape) if t.format.mode_ordering == tuple(range(t.order)) \
        else to_torch(t)
    if tuple(order) != tuple(range(t.order)):
        x = x.permute(*order)
    x = x.contiguous()
    # torch calls a permuted view with size-1 dims contiguous without fixing their strides;
    # the kernels read the innermost stride, so give every dim its canonical stride
    want, acc = [], 1
    for d in reversed(x.shape):
        want.append(acc)
        acc *= d
    if tuple(reversed(want)) != x.stride():
        x = x.clone(memory_format=torch.contiguous_format)
    return x


def _dense_result(name: str, arr: torch.Tensor) -> Tensor:
    fmt = dense_format(tuple(arr.shape))
    st = TensorStorage(fmt, tuple(DenseLevel(s) for s in arr.shape),
                       arr.reshape(-1).to(VALUE_DTYPE).contiguous())
    return Tensor(name, tuple(arr.shape), st)


def _compressed_dense_result(name, shape, rows: torch.Tensor, values: torch.Tensor) -> Tensor:
    """[compressed(rows), dense] 2-D result (the workspace-drained output)."""
    n = rows.numel()
    pos = torch.tensor([0, n], dtype=torch.int32, device=values.device)
    fmt = TensorFormat(shape, (0, 1), (LevelFormat.COMPRESSED, LevelFormat.DENSE))
    st = TensorStorage(fmt, (CompressedLevel(pos, rows.to(torch.int32).contiguous()),
                             DenseLevel(shape[1])), values.reshape(-1).contiguous())
    return Tensor(name, tuple(shape), st)


def _n_blocks(extent: int, sched: Schedule, var) -> int:
    if sched.tile_size is None or var not in sched.tiles:
        return 0
    return -(-extent // sched.tile_size)


class _Ctx:
    def __init__(self, sched: Schedule, bindings, out_fmt: TensorFormat, variant: str | None):
        self.sched = sched
        self.expr: TensorExpr = sched.expr
        self.out_fmt = out_fmt
        self.variant = variant
        self.counter = OpCounter()
        self.extents = index_extents(self.expr)
        self.tensor_of: dict[int, Tensor] = {}
        for a in self.expr.accesses:
            t = a.tensor
            if bindings is not None and a.tensor.name in bindings:
                t = bindings[a.tensor.name]
                if t.shape != a.tensor.shape or t.format != a.tensor.format:
                    raise ShapeError(
                        f"rebinding of {a.tensor.name} must match the scheduled shape and format")
            self.tensor_of[id(a)] = t
        self.chosen: list[str] = []

    def t(self, a: Access) -> Tensor:
        return self.tensor_of[id(a)]


# ---------------------------------------------------------------------------
# Term matchers
# ---------------------------------------------------------------------------


@dataclass
class _SpmmTerm:
    A: Access          # 2-D sparse
    B: Access          # 1-D or 2-D dense
    i: object
    j: object
    k: object | None   # None for SpMV


def _match_spmm(term, out_vars) -> _SpmmTerm | None:
    if len(term) != 2:
        return None
    sp = [a for a in term if a.tensor.format.has_sparse_levels]
    dn = [a for a in term if not a.tensor.format.has_sparse_levels]
    if len(sp) != 1 or len(dn) != 1:
        return None
    A, B = sp[0], dn[0]
    if A.tensor.order != 2 or B.tensor.order not in (1, 2):
        return None
    shared = set(A.indices) & set(B.indices)
    if len(shared) != 1:
        return None
    j = next(iter(shared))
    if j in out_vars:
        return None
    i = A.indices[0] if A.indices[1] == j else A.indices[1]
    k = None
    if B.tensor.order == 2:
        k = B.indices[0] if B.indices[1] == j else B.indices[1]
        if k == i:
            return None
    want = {i} if k is None else {i, k}
    if set(out_vars) != want:
        return None
    return _SpmmTerm(A, B, i, j, k)


@dataclass
class _SddmmTerm:
    M: Access
    Q: Access
    K: Access
    h: object | None
    i: object
    j: object
    d: object


def _match_sddmm(term, out_vars) -> _SddmmTerm | None:
    if len(term) != 3:
        return None
    sp = [a for a in term if a.tensor.format.has_sparse_levels]
    dn = [a for a in term if not a.tensor.format.has_sparse_levels]
    if len(sp) != 1 or len(dn) != 2 or sp[0].tensor.order != 2:
        return None
    M = sp[0]
    i, j = M.indices
    red = {v for a in term for v in a.indices} - set(out_vars)
    if len(red) != 1:
        return None
    d = next(iter(red))
    h = None
    extra = [v for v in out_vars if v not in (i, j)]
    if len(extra) == 1:
        h = extra[0]
    elif extra:
        return None
    want = (i, j) if h is None else (h, i, j)
    if tuple(out_vars) != want:
        return None
    Q = K = None
    for a in dn:
        s = set(a.indices)
        hs = {h} if h is not None else set()
        if s == {i, d} | hs:
            Q = a
        elif s == {j, d} | hs:
            K = a
    if Q is None or K is None:
        return None
    return _SddmmTerm(M, Q, K, h, i, j, d)


@dataclass
class _MttkrpTerm:
    T: Access
    B: Access
    C: Access
    i: object
    j: object
    k: object
    r: object
    b_first: bool


def _match_mttkrp(term, out_vars) -> _MttkrpTerm | None:
    """MTTKRP in any mode: M(i,r) = T(..i..) * B(j,r) * C(k,r), i one of T's indices
    (CP-ALS runs all three modes). ``i`` is the output mode, ``j``/``k`` the other two
    in T's index order."""
    if len(term) != 3 or len(out_vars) != 2:
        return None
    sp = [a for a in term if a.tensor.format.has_sparse_levels]
    if len(sp) != 1 or sp[0].tensor.order != 3:
        return None
    T = sp[0]
    i, r = out_vars
    if i not in T.indices or r in T.indices:
        return None
    j, k = (v for v in T.indices if v != i)
    dn = [a for a in term if a is not T]
    if any(a.tensor.format.has_sparse_levels or a.tensor.order != 2 for a in dn):
        return None
    Bs = [a for a in dn if set(a.indices) == {j, r}]
    Cs = [a for a in dn if set(a.indices) == {k, r}]
    if len(Bs) != 1 or len(Cs) != 1:
        return None
    b_first = term.index(Bs[0]) < term.index(Cs[0])
    return _MttkrpTerm(T, Bs[0], Cs[0], i, j, k, r, b_first)


@dataclass
class _BatchedPvTerm:
    P: Access
    V: Access
    h: object
    i: object
    j: object
    d: object


def _match_batched_pv(term, out_vars) -> _BatchedPvTerm | None:
    if len(term) != 2 or len(out_vars) != 3:
        return None
    sp = [a for a in term if a.tensor.format.has_sparse_levels]
    if len(sp) != 1 or sp[0].tensor.order != 3:
        return None
    P = sp[0]
    V = term[1] if term[0] is P else term[0]
    if V.tensor.format.has_sparse_levels or V.tensor.order != 3:
        return None
    h, i, j = P.indices
    d = next((v for v in V.indices if v not in (h, j)), None)
    if d is None or set(V.indices) != {h, j, d} or tuple(out_vars) != (h, i, d):
        return None
    f = P.tensor.format
    if f.mode_ordering != (0, 1, 2) or f.levels != (
            LevelFormat.DENSE, LevelFormat.DENSE, LevelFormat.COMPRESSED):
        return None
    return _BatchedPvTerm(P, V, h, i, j, d)


# ---------------------------------------------------------------------------
# Term executors
# ---------------------------------------------------------------------------


def _spmm_rows(ctx: _Ctx, m: _SpmmTerm, addend: torch.Tensor | None = None, relu=False):
    """Run one SpMM term; returns (view, Y) with Y rows = view segments (or all rows)."""
    A = ctx.t(m.A)
    B = ctx.t(m.B)
    row_dim = m.A.indices.index(m.i)
    view = row_view(A, row_dim)
    if m.k is None:
        Bd = _dense_torch(B, (0,)).reshape(-1, 1)
    else:
        Bd = _dense_torch(B, (m.B.indices.index(m.j), m.B.indices.index(m.k)))
    K = Bd.shape[1]
    key = (row_dim,)
    stats = _stats(A, view, key)
    variant = ctx.variant or ops.choose_variant(stats, K, aligned=(K % 4 == 0), n_cols=Bd.shape[0])
    if variant not in ("row", "merge", "coltile"):
        raise ValueError(f"unknown variant {variant!r}")
    partition = None
    if variant == "merge":
        partition = _partition(A, view, key, K)
    elif variant == "coltile":
        partition = _cache(A, ("coltile",) + key,
                           lambda: ops.coltile_plan(view.rowptr, view.cols, Bd.shape[0], view.vals))
    if addend is not None and not view.dense_rows:
        raise UnsupportedExpressionError("dense addend with a compressed row level")
    Y = ops.spmm_csr(view.rowptr, view.cols, view.vals, Bd, addend=addend, relu=relu,
                     variant=variant, partition=partition, stats=stats)
    ctx.chosen.append(f"spmm:{variant}:{view.kind}")
    return view, Y, K


def _spmm_counters(ctx: _Ctx, m: _SpmmTerm, view: RowView, K: int):
    nnz = view.vals.numel()
    if m.k is None:  # SpMV: scalar path (engine.py:515-531 not taken)
        if view.kind == "csr":
            ctx.counter.add(nnz, nnz + view.n_rows, 2 * nnz)
        elif view.kind in ("coo", "dcsr"):  # workspace per distinct row
            ctx.counter.add(nnz, nnz + view.n_segments, 3 * view.n_segments + 2 * nnz)
        else:  # column-major storage walked [j, i]
            ctx.counter.add(nnz, nnz, 2 * nnz)
        return
    order = ctx.sched.loop_order
    nblk = _n_blocks(K, ctx.sched, m.k)
    if view.kind == "csr" and order.index(m.i) < order.index(m.k):
        # dense output, vectorised tail over k (engine.py:512-565)
        it = nnz * K + 2 * nnz * max(nblk, 1) + nblk
        ctx.counter.add(nnz * K, nnz * K, it)
    elif view.kind == "csr":
        # output spelled (k, i): order [k, i, j], scalar sink per (k, i)
        ctx.counter.add(nnz * K, nnz * K + K * view.n_rows, 2 * nnz * K)
    elif view.kind in ("coo", "dcsr"):
        n_seg = view.n_segments
        it = nblk * (1 + 2 * n_seg + 2 * nnz) if nblk else 3 * n_seg + 2 * nnz
        ctx.counter.add(nnz * K, nnz * K, it)
    else:  # column-major storage walked [j, i, k]
        ctx.counter.add(nnz * K, nnz * K, max(nblk, 1) * (1 + 2 * nnz) if nblk else 2 * nnz)


def _exec_dense_output(ctx: _Ctx) -> Tensor:
    """Dense output: every term is an SpMM-like term or all-dense; accumulate."""
    e = ctx.expr
    out_vars = e.output_indices
    ext = ctx.extents
    out_shape = tuple(ext[v] for v in out_vars)
    if ctx.out_fmt.mode_ordering != tuple(range(len(out_vars))):
        raise UnsupportedExpressionError("dense outputs with a permuted mode ordering")
    terms = e.terms()
    acc: torch.Tensor | None = None
    dev = next(iter(ctx.tensor_of.values())).device
    for term in terms:
        m = _match_spmm(term, out_vars)
        if m is not None:
            A = ctx.t(m.A)
            row_dim = m.A.indices.index(m.i)
            view = row_view(A, row_dim)
            ik_order = m.k is None or list(out_vars) == [m.i, m.k]
            use_addend = acc is not None and view.dense_rows and ik_order
            view, Y, K = _spmm_rows(ctx, m, addend=acc if use_addend else None)
            _spmm_counters(ctx, m, view, K)
            if not view.dense_rows:
                full = torch.zeros((view.n_rows, K), dtype=torch.float32, device=Y.device)
                full.index_copy_(0, view.seg_rows.long(), Y)
                Y = full
            res = Y.reshape(out_shape) if m.k is None else (Y if ik_order else Y.t())
            if use_addend:
                acc = res
            else:
                acc = res.contiguous() if acc is None else acc + res
            continue
        pv = _match_batched_pv(term, out_vars)
        if pv is not None:
            res = _exec_batched_pv(ctx, pv)
            acc = res if acc is None else acc + res
            continue
        if all(not a.tensor.format.has_sparse_levels for a in term):
            res = _dense_einsum(ctx, term, out_vars)
            # dense addend term: adds m*K (+ block advances when k is tiled)
            n_out = math.prod(out_shape)
            nblk = _n_blocks(out_shape[-1], ctx.sched, out_vars[-1]) if out_vars else 0
            ctx.counter.add(0, n_out, n_out + nblk)
            acc = res if acc is None else acc + res
            continue
        raise UnsupportedExpressionError(
            "no device kernel for term " + " * ".join(f"{a.name}({','.join(v.name for v in a.indices)})"
                                                        for a in term))
    if acc is None:
        acc = torch.zeros(out_shape, dtype=torch.float32, device=dev)
    return _dense_result(e.output_name, acc.reshape(out_shape))


def _dense_einsum(ctx: _Ctx, term, out_vars) -> torch.Tensor:
    """One all-dense term over the output's index space. Output indices the term does
    not mention are broadcast (the reference's eval_dense adds the term's value at
    every such coordinate, oracle.py:35-46)."""
    letters = {}
    for v in list(out_vars) + [v for a in term for v in a.indices]:
        letters.setdefault(v, string.ascii_letters[len(letters)])
    term_vars = {v for a in term for v in a.indices}
    present = [v for v in out_vars if v in term_vars]
    subs = ",".join("".join(letters[v] for v in a.indices) for a in term)
    eq = f"{subs}->{''.join(letters[v] for v in present)}"
    ops_ = [_dense_torch(ctx.t(a), tuple(range(a.tensor.order))) for a in term]
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        r = torch.einsum(eq, *ops_).to(torch.float32)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    if len(present) != len(out_vars):
        shape = [ctx.extents[v] if v in term_vars else 1 for v in out_vars]
        r = r.reshape(shape).expand(*[ctx.extents[v] for v in out_vars]).contiguous()
    return r


def _exec_batched_pv(ctx: _Ctx, pv: _BatchedPvTerm) -> torch.Tensor:
    P = ctx.t(pv.P)
    V = ctx.t(pv.V)
    H, m, n = P.shape
    Vd = _dense_torch(V, (pv.V.indices.index(pv.h), pv.V.indices.index(pv.j), pv.V.indices.index(pv.d)))
    d = Vd.shape[2]
    shared = P._cache.get("shared_pattern")
    L = P.storage.levels[2]
    nnz_total = L.crd.numel()
    if shared is not None:
        rowptr, colidx = shared
        vals = P.storage.values.reshape(H, -1)
        stats = _cache(P, ("stats", "shared"), lambda: ops.row_stats(rowptr))
        variant = ctx.variant if ctx.variant in ("row", "merge") else (
            "merge" if stats.skew > ops.MERGE_SKEW_THRESHOLD else "row")
        part = _cache(P, ("partition", "shared"), lambda: ops.merge_partition(rowptr, colidx.numel(), k=d, batch=H)) \
            if variant == "merge" else None
        O = ops.spmm_csr_batched(rowptr, colidx, vals, Vd, variant=variant, partition=part, stats=stats)
        ctx.chosen.append(f"pv:batched-{variant}")
    else:
        # per-head structures differ: one CSR over H*m rows gathering from V viewed as (H*n, d)
        def build():
            pos = L.pos
            per_row = (pos[1:] - pos[:-1]).long()
            head_of_row = torch.arange(H * m, device=pos.device) // m
            off = torch.repeat_interleave(head_of_row * n, per_row)
            return (L.crd.long() + off).to(torch.int32)

        cols = _cache(P, ("pv_cols",), build)
        stats = _cache(P, ("stats", "flat"), lambda: ops.row_stats(L.pos))
        variant = ctx.variant if ctx.variant in ("row", "merge") else ops.choose_variant(stats, d)
        if variant == "coltile":
            variant = "merge"
        part = _cache(P, ("partition", "flat"), lambda: ops.merge_partition(L.pos, nnz_total, k=d)) \
            if variant == "merge" else None
        O = ops.spmm_csr(L.pos, cols, P.storage.values, Vd.reshape(H * n, d), variant=variant,
                         partition=part, stats=stats).reshape(H, m, d)
        ctx.chosen.append(f"pv:flat-{variant}")
    nblk = _n_blocks(d, ctx.sched, pv.d)
    ctx.counter.add(nnz_total * d, nnz_total * d, nnz_total * d + 2 * nnz_total * max(nblk, 1) + nblk)
    return O


def _exec_sddmm(ctx: _Ctx, s: _SddmmTerm) -> Tensor:
    M = ctx.t(s.M)
    if s.M.indices != (s.i, s.j):
        raise UnsupportedExpressionError("SDDMM output must list the mask's indices in order")
    view = row_view(M, 0)
    hs = () if s.h is None else (s.h,)
    Qd = _dense_torch(ctx.t(s.Q), tuple(s.Q.indices.index(v) for v in hs + (s.i, s.d)))
    Kd = _dense_torch(ctx.t(s.K), tuple(s.K.indices.index(v) for v in hs + (s.j, s.d)))
    d = Qd.shape[-1]
    if d <= 128:
        dk = next(w for w in (4, 8, 16, 32, 64, 128) if w >= d)
        if dk != d:  # zero-pad the reduction dim to the kernel's lane width (exact: adds 0 products)
            Qd = torch.nn.functional.pad(Qd, (0, dk - d))
            Kd = torch.nn.functional.pad(Kd, (0, dk - d))
        vals = ops.sddmm_csr(view.rowptr, view.cols, Qd, Kd, maskvals=view.vals, scale=1.0)
    else:
        # wider reductions: 128-wide blocks of the kernel summed left to right (the reference's
        # tiled d-blocks), then the mask value, as in the reference (dot first, times m_ij)
        vals = None
        for c0 in range(0, d, 128):
            w = min(128, d - c0)
            dk = next(x for x in (4, 8, 16, 32, 64, 128) if x >= w)
            Qc, Kc = Qd[..., c0:c0 + w], Kd[..., c0:c0 + w]
            if dk != w:
                Qc = torch.nn.functional.pad(Qc, (0, dk - w))
                Kc = torch.nn.functional.pad(Kc, (0, dk - w))
            # (a fresh copy: canonical strides even for size-1 dims of the sliced operands)
            Qc = Qc.clone(memory_format=torch.contiguous_format)
            Kc = Kc.clone(memory_format=torch.contiguous_format)
            part = ops.sddmm_csr(view.rowptr, view.cols, Qc, Kc, scale=1.0)
            vals = part if vals is None else vals + part
        vals = vals * view.vals
    ctx.chosen.append(f"sddmm:{view.kind}")
    nnz = view.vals.numel()
    H = 1 if s.h is None else Qd.shape[0]
    n_rows = M.shape[0]
    nblk = _n_blocks(d, ctx.sched, s.d)
    tot = H * nnz
    ctx.counter.add(tot * (d + 1), tot * (d + 1),
                    tot * d + (3 + nblk) * tot + H * n_rows + (H if s.h is not None else 0))
    fmt = ctx.out_fmt
    if s.h is None:
        if view.kind == "csr" and fmt.levels == (LevelFormat.DENSE, LevelFormat.COMPRESSED):
            levels = (DenseLevel(n_rows), CompressedLevel(view.rowptr, view.cols))
        elif view.kind in ("dcsr", "coo", "sorted") and fmt.levels == (
                LevelFormat.COMPRESSED, LevelFormat.COMPRESSED):
            n_seg = view.n_segments
            top = torch.tensor([0, n_seg], dtype=torch.int32, device=vals.device)
            levels = (CompressedLevel(top, view.seg_rows), CompressedLevel(view.rowptr, view.cols))
        else:
            coords, _ = stored_entries_torch(M)
            return _assemble(M.shape, fmt, coords, vals.reshape(-1)[_view_perm(M, view)], ctx.expr.output_name)
        st = TensorStorage(fmt, levels, vals.reshape(-1))
        return Tensor(ctx.expr.output_name, M.shape, st)
    # multi-head: [dense h, dense i, compressed j], the mask's pattern per head
    if view.kind != "csr" or fmt.levels != (LevelFormat.DENSE, LevelFormat.DENSE, LevelFormat.COMPRESSED):
        raise UnsupportedExpressionError("multi-head SDDMM needs a CSR mask and a [dense,dense,compressed] output")
    rp = view.rowptr.long()
    pos = torch.cat([(rp[:-1][None, :] + torch.arange(H, device=rp.device)[:, None] * nnz).reshape(-1),
                     torch.tensor([H * nnz], device=rp.device)]).to(torch.int32)
    crd = view.cols.repeat(H)
    shape = (H,) + M.shape
    st = TensorStorage(fmt, (DenseLevel(H), DenseLevel(n_rows), CompressedLevel(pos, crd)), vals.reshape(-1))
    out = Tensor(ctx.expr.output_name, shape, st)
    out._cache["shared_pattern"] = (view.rowptr, view.cols)
    return out


def _view_perm(t: Tensor, view: RowView) -> torch.Tensor:
    """Permutation from stored order to the view's (row, col) order (identity for CSR/DCSR/COO)."""
    n = view.vals.numel()
    if view.kind != "sorted":
        return torch.arange(n, device=view.vals.device)
    coords, _ = stored_entries_torch(t)
    key = coords[:, 0] * t.shape[1] + coords[:, 1]
    order = torch.sort(key, stable=True).indices
    inv = torch.empty_like(order)
    inv[order] = torch.arange(n, device=order.device)
    return inv


def _exec_mttkrp(ctx: _Ctx, mk: _MttkrpTerm) -> Tensor:
    T = ctx.t(mk.T)
    f = T.format
    if not f.is_coordinate:
        raise UnsupportedExpressionError("MTTKRP needs a COO tensor")
    if ctx.out_fmt.levels != (LevelFormat.COMPRESSED, LevelFormat.DENSE) or ctx.out_fmt.mode_ordering != (0, 1):
        raise UnsupportedExpressionError("MTTKRP output must be [compressed, dense]")
    # the kernel walks entries sorted by (output mode, j, k): for another output mode (or
    # another storage order) a device re-sorted COO view of T is built once and cached
    order = tuple(mk.T.indices.index(v) for v in (mk.i, mk.j, mk.k))
    view = T if f.mode_ordering == order else _cache(
        T, ("mttkrp_view", order), lambda: convert(T, f.with_mode_ordering(order)))
    st = view.storage
    # op counters follow the reference, which walks T in its storage order for every mode
    base = T.storage if f.mode_ordering == (0, 1, 2) else _cache(
        T, ("mttkrp_view", (0, 1, 2)), lambda: convert(T, f.with_mode_ordering((0, 1, 2)))).storage
    seg = _cache(view, ("coo_segments",), lambda: ops.coo_segments(st.levels[0].crd))
    Bd = _dense_torch(ctx.t(mk.B), (mk.B.indices.index(mk.j), mk.B.indices.index(mk.r)))
    Cd = _dense_torch(ctx.t(mk.C), (mk.C.indices.index(mk.k), mk.C.indices.index(mk.r)))
    if not mk.b_first:
        # (t*C)*B order: swap the gathered operands and their coordinate columns
        jc, kc, Bd, Cd = st.levels[2].crd, st.levels[1].crd, Cd, Bd
    else:
        jc, kc = st.levels[1].crd, st.levels[2].crd
    variant = ctx.variant if ctx.variant in ("row", "merge") else "merge"
    fkey = (Bd.shape[0], Bd.stride(0), Cd.shape[0], Cd.stride(0))
    # the plan holds the entries as prepared items for these factor shapes (jc/kc swapped with B/C above)
    part = _cache(view, ("partition", "mttkrp", Bd.shape[1], mk.b_first, fkey),
                  lambda: ops.merge_partition(seg.ptr, st.values.numel(), k=Bd.shape[1], kind="mttkrp",
                                              jcrd=jc, kcrd=kc, vals=st.values, factors=fkey)) \
        if variant == "merge" else None
    M = ops.mttkrp_coo3(seg, jc, kc, st.values, Bd, Cd, variant=variant, partition=part)
    ctx.chosen.append(f"mttkrp:{variant}")
    nnz = st.values.numel()
    R = Bd.shape[1]
    nblk = _n_blocks(R, ctx.sched, mk.r)

    def distinct_prefix(levels):
        c0 = base.levels[0].crd
        if nnz == 0:
            return 0
        new = torch.zeros(nnz, dtype=torch.bool, device=c0.device)
        new[0] = True
        for lv in base.levels[:levels]:
            new[1:] |= lv.crd[1:] != lv.crd[:-1]
        return int(new.sum().item())

    n_i = seg.n_seg if base is st else _cache(T, ("distinct_i",), lambda: distinct_prefix(1))
    n_ij = _cache(T, ("distinct_ij",), lambda: distinct_prefix(2))
    body = 2 * n_i + 2 * n_ij + 2 * nnz
    ctx.counter.add(2 * nnz * R, nnz * R, nblk * (1 + body) if nblk else body + n_i)
    return _compressed_dense_result(ctx.expr.output_name, (T.shape[mk.T.indices.index(mk.i)], R), seg.rows, M)


def _exec_sparse_spmm(ctx: _Ctx, m: _SpmmTerm) -> Tensor:
    """SpMM whose inferred output is [compressed i, dense k] (COO / DCSR / CSC operands)."""
    out_vars = ctx.expr.output_indices
    if m.k is None:
        return _exec_sparse_spmv(ctx, m)
    if list(out_vars) != [m.i, m.k]:
        raise UnsupportedExpressionError("sparse-output SpMM must be spelled C(i,k)")
    if ctx.out_fmt.levels != (LevelFormat.COMPRESSED, LevelFormat.DENSE) or \
            ctx.out_fmt.mode_ordering != (0, 1):
        raise UnsupportedExpressionError(
            f"SpMM into {ctx.out_fmt.name()} is not supported on the device (dense or "
            "[compressed, dense] outputs only)")
    view, Y, K = _spmm_rows(ctx, m)
    _spmm_counters(ctx, m, view, K)
    if view.dense_rows:
        # compressed i-level over a CSR view: keep rows that hold entries
        lens = view.rowptr[1:] - view.rowptr[:-1]
        rows = torch.nonzero(lens > 0).flatten().to(torch.int32)
        Y = Y[rows.long()]
    else:
        rows = view.seg_rows
    return _compressed_dense_result(ctx.expr.output_name, (view.n_rows, K), rows, Y)


def _exec_sparse_spmv(ctx: _Ctx, m: _SpmmTerm) -> Tensor:
    """SpMV whose inferred output is a compressed vector over the rows that hold entries
    (COO / DCSR / CSC operands; the reference's 1-D workspace drain)."""
    if ctx.out_fmt.levels != (LevelFormat.COMPRESSED,):
        raise UnsupportedExpressionError(f"SpMV into {ctx.out_fmt.name()} is not supported on the device")
    view, Y, K = _spmm_rows(ctx, m)
    _spmm_counters(ctx, m, view, K)
    if view.dense_rows:
        lens = view.rowptr[1:] - view.rowptr[:-1]
        rows = torch.nonzero(lens > 0).flatten().to(torch.int32)
        Y = Y[rows.long()]
    else:
        rows = view.seg_rows
    n = rows.numel()
    pos = torch.tensor([0, n], dtype=torch.int32, device=Y.device)
    st_ = TensorStorage(ctx.out_fmt, (CompressedLevel(pos, rows.to(torch.int32).contiguous()),),
                        Y.reshape(-1).contiguous())
    return Tensor(ctx.expr.output_name, (view.n_rows,), st_)


# ---------------------------------------------------------------------------
# Sparse x sparse
# ---------------------------------------------------------------------------


def _is_csr(t: Tensor) -> bool:
    f = t.format
    return f.order == 2 and f.mode_ordering == (0, 1) and f.levels == (LevelFormat.DENSE, LevelFormat.COMPRESSED)


def _csr_out(ctx: _Ctx, shape, r: ops.CsrResult) -> Tensor:
    fmt = ctx.out_fmt
    if fmt.order != 2 or fmt.mode_ordering != (0, 1) or fmt.levels != (LevelFormat.DENSE, LevelFormat.COMPRESSED):
        raise UnsupportedExpressionError(
            f"sparse x sparse into {fmt.name()} is not supported on the device (CSR output only)")
    st = TensorStorage(fmt, (DenseLevel(shape[0]), CompressedLevel(r.rowptr, r.colidx)), r.vals)
    return Tensor(ctx.expr.output_name, tuple(shape), st)


@dataclass
class _SpgemmTerm:
    A: Access
    B: Access


def _match_spgemm(term, out_vars) -> _SpgemmTerm | None:
    if len(term) != 2 or not all(a.tensor.format.has_sparse_levels and a.tensor.order == 2 for a in term):
        return None
    for A, B in ((term[0], term[1]), (term[1], term[0])):
        i, j = A.indices
        j2, k = B.indices
        if j == j2 and len({i, j, k}) == 3 and list(out_vars) == [i, k]:
            return _SpgemmTerm(A, B)
    return None


def _exec_spgemm(ctx: _Ctx, g: _SpgemmTerm) -> Tensor:
    """Gustavson SpGEMM; counters of the reference's [i, j, k] workspace nest:
    mults = adds = P (products), iterator advances = m + 2 nnz(A) + 2 P."""
    A, B = ctx.t(g.A), ctx.t(g.B)
    if not (_is_csr(A) and _is_csr(B)):
        raise UnsupportedExpressionError("device SpGEMM needs CSR operands accessed in storage order")
    la, lb = A.storage.levels[1], B.storage.levels[1]
    r = ops.spgemm_csr(la.pos, la.crd, A.storage.values, lb.pos, lb.crd, B.storage.values, B.shape[1])
    ctx.chosen.append("spgemm:dense-window" if B.shape[1] <= 6144 else "spgemm:esc")
    m, nnz_a = A.shape[0], int(A.storage.values.numel())
    ctx.counter.add(r.products, r.products, m + 2 * nnz_a + 2 * r.products)
    return _csr_out(ctx, (A.shape[0], B.shape[1]), r)


def _match_ewise(terms, out_vars):
    """("add", A, B) for A(i,j) + B(i,j); ("mul", A, B) for A(i,j) * B(i,j)."""
    ov = tuple(out_vars)

    def ok(a):
        return a.tensor.format.has_sparse_levels and a.tensor.order == 2 and a.indices == ov
    if len(terms) == 2 and all(len(t) == 1 and ok(t[0]) for t in terms):
        return "add", terms[0][0], terms[1][0]
    if len(terms) == 1 and len(terms[0]) == 2 and all(ok(a) for a in terms[0]):
        return "mul", terms[0][0], terms[0][1]
    return None


def _exec_ewise(ctx: _Ctx, op: str, a: Access, b: Access) -> Tensor:
    """Element-wise union / intersection; counters of the reference's co-iteration
    (`_union_sorted` / `_intersect_sorted` over [i, j], engine.py:208-230, 577-644)."""
    A, B = ctx.t(a), ctx.t(b)
    if not (_is_csr(A) and _is_csr(B)):
        raise UnsupportedExpressionError("device element-wise ops need CSR operands accessed in storage order")
    la, lb = A.storage.levels[1], B.storage.levels[1]
    r = ops.csr_ewise(op, la.pos, la.crd, A.storage.values, lb.pos, lb.crd, B.storage.values)
    ctx.chosen.append(f"ewise:{op}")
    m = A.shape[0]
    nnz_a, nnz_b, nnz_c = int(A.storage.values.numel()), int(B.storage.values.numel()), int(r.vals.numel())
    if op == "add":
        ctx.counter.add(0, nnz_a + nnz_b, m + 2 * (nnz_a + nnz_b) + 2 * nnz_c)
    else:
        lens = torch.minimum(la.pos[1:] - la.pos[:-1], lb.pos[1:] - lb.pos[:-1]).long()
        both = int((lens > 0).sum().item())
        ctx.counter.add(nnz_c, nnz_c, m + int(lens.sum().item()) + both + 4 * nnz_c)
    return _csr_out(ctx, A.shape, r)


def _dispatch(ctx: _Ctx) -> Tensor:
    """Dedicated kernel when the expression matches one; otherwise the device loop-nest
    walker (`generic.py`), which follows the reference interpreter's iteration space."""
    e = ctx.expr
    if ctx.out_fmt.shape != e.output_shape:
        raise ShapeError(f"output format shape {ctx.out_fmt.shape} != expression output {e.output_shape}")
    _require_device(ctx.tensor_of.values())
    try:
        return _dispatch_kernels(ctx)
    except UnsupportedExpressionError as err:
        ctx.counter = OpCounter()
        ctx.chosen = [f"generic:device-walk ({err})"[:160]]
        try:
            return execute_generic(ctx.sched, ctx.tensor_of, ctx.out_fmt, ctx.counter)
        except TooLargeForGenericWalk as big:
            raise UnsupportedExpressionError(f"{err}; generic walk: {big}") from None


def _dispatch_kernels(ctx: _Ctx) -> Tensor:
    e = ctx.expr
    out_fmt = ctx.out_fmt
    terms = e.terms()
    out_vars = e.output_indices
    if not out_fmt.has_sparse_levels:
        return _exec_dense_output(ctx)
    if len(terms) == 1:
        term = terms[0]
        s = _match_sddmm(term, out_vars)
        if s is not None:
            return _exec_sddmm(ctx, s)
        mk = _match_mttkrp(term, out_vars)
        if mk is not None:
            return _exec_mttkrp(ctx, mk)
        sp = _match_spmm(term, out_vars)
        if sp is not None:
            return _exec_sparse_spmm(ctx, sp)
        g = _match_spgemm(term, out_vars)
        if g is not None:
            return _exec_spgemm(ctx, g)
    ew = _match_ewise(terms, out_vars)
    if ew is not None:
        return _exec_ewise(ctx, *ew)
    raise UnsupportedExpressionError(
        f"no device kernel for {e.output_name} with output format {out_fmt.name()} "
        "(supported sparse outputs: SDDMM, MTTKRP, COO/DCSR/CSC SpMM, CSR SpGEMM, CSR + CSR, CSR .* CSR)")


# ---------------------------------------------------------------------------
# Public entry points (`engine.py:657-724`)
# ---------------------------------------------------------------------------


def execute(sched: Schedule, bindings: dict | None = None, out_fmt: TensorFormat | None = None,
            variant: str | None = None):
    """Run a schedule on the GPU; returns ``(Tensor, OpCounter)``.

    ``variant`` overrides the kernel-variant choice ("row", "merge",
    "coltile") for SpMM-shaped terms.
    """
    out_fmt = out_fmt if out_fmt is not None else sched.out_format
    fast = _fast_spmm_plan(sched, out_fmt)
    if fast is not None:
        got = _fast_spmm(sched, fast, bindings, variant)
        if got is not None:
            return got
    if set(sched.loop_order) != set(get_index_variables(sched.expr)):
        raise ValueError("schedule does not cover the expression's index variables")
    ctx = _Ctx(sched, bindings, out_fmt, variant)
    result = _dispatch(ctx)
    execute.last_variants = tuple(ctx.chosen)
    return result, ctx.counter


# ---- repeated calls of the hot path --------------------------------------------------
# A schedule whose expression is one CSR SpMM / SpMV term into a dense output is
# recognised once (structure only, cached on the schedule); later calls look up the
# operands' cached row view / statistics / partition and launch directly. Same kernels,
# arguments, counters and result as the general dispatch below.


@dataclass
class _FastSpmm:
    m: _SpmmTerm
    a_name: str
    b_name: str
    b_order: tuple
    out_shape: tuple
    ik_order: bool


def _fast_spmm_plan(sched: Schedule, out_fmt: TensorFormat):
    cache = sched.__dict__.setdefault("_fast", {})
    if out_fmt in cache:
        return cache[out_fmt]
    plan = None
    e = sched.expr
    terms = e.terms()
    out_vars = e.output_indices
    if (len(terms) == 1 and not out_fmt.has_sparse_levels and out_fmt.shape == e.output_shape
            and out_fmt.mode_ordering == tuple(range(len(out_vars)))
            and set(sched.loop_order) == set(get_index_variables(e))):
        m = _match_spmm(terms[0], out_vars)
        if m is not None:
            f = m.A.tensor.format
            row_dim = m.A.indices.index(m.i)
            csr_like = f.mode_ordering[0] == row_dim and f.levels == (LevelFormat.DENSE, LevelFormat.COMPRESSED)
            if csr_like and m.A.tensor.name != m.B.tensor.name:
                b_order = (0,) if m.k is None else (m.B.indices.index(m.j), m.B.indices.index(m.k))
                ext = index_extents(e)
                plan = _FastSpmm(m, m.A.tensor.name, m.B.tensor.name, b_order,
                                 tuple(ext[v] for v in out_vars), m.k is None or list(out_vars) == [m.i, m.k])
    cache[out_fmt] = plan
    return plan


class _LightCtx:
    def __init__(self, sched, variant, A, B, m):
        self.sched, self.variant, self.counter, self.chosen = sched, variant, OpCounter(), []
        self._t = {id(m.A): A, id(m.B): B}

    def t(self, a: Access) -> Tensor:
        return self._t[id(a)]


def _fast_spmm(sched: Schedule, f: _FastSpmm, bindings, variant):
    m = f.m
    A, B = m.A.tensor, m.B.tensor
    if bindings:
        A = bindings.get(f.a_name, A)
        B = bindings.get(f.b_name, B)
        for t, a in ((A, m.A), (B, m.B)):
            if t is not a.tensor and (t.shape != a.tensor.shape or t.format != a.tensor.format):
                raise ShapeError(f"rebinding of {a.tensor.name} must match the scheduled shape and format")
    if not (A.storage.values.is_cuda and B.storage.values.is_cuda):
        return None  # the general path raises the device error
    ctx = _LightCtx(sched, variant, A, B, m)
    view, Y, K = _spmm_rows(ctx, m)
    _spmm_counters(ctx, m, view, K)
    res = Y.reshape(f.out_shape) if m.k is None else (Y if f.ik_order else Y.t().contiguous())
    execute.last_variants = tuple(ctx.chosen)
    return _dense_result(sched.expr.output_name, res), ctx.counter


execute.last_variants = ()


def run_with_report(e: TensorExpr, bindings: dict | None = None, out_format: TensorFormat | None = None,
                    tile_size: int = DEFAULT_TILE_SIZE, tiling: bool = True,
                    weights: CostModel = CostModel(), variant: str | None = None):
    """Plan + execute with a JSON-ready report (`engine.py:667-717`).

    All-dense expressions take the dense path (torch/cuBLAS, TF32 off, the
    paper's "dense -> torch" branch); everything else is inferred, scheduled,
    tiled and dispatched to a kernel variant. ``wall_time_ns`` brackets the
    launch and a device synchronisation.
    """
    if bindings:
        for a in e.accesses:
            t = bindings.get(a.tensor.name)
            if t is not None and t.shape != a.tensor.shape:
                raise ShapeError(f"binding for {a.tensor.name} has shape {t.shape}")
    if all(not a.tensor.format.has_sparse_levels for a in e.accesses):
        return _run_dense(e, bindings, out_format, weights, timed=True)

    out_fmt, sched = _plan(e, out_format, tile_size, tiling, weights)
    t0 = time.perf_counter_ns()
    result, counter = execute(sched, bindings, variant=variant)
    torch.cuda.synchronize()
    wall = time.perf_counter_ns() - t0
    report = {
        "path": "sparse",
        "inferred_format": infer_format(e).name(),
        "out_format": out_fmt.name(),
        "schedule": schedule_to_dict(sched),
        "counters": counter.as_dict(),
        "wall_time_ns": wall,
        "variants": list(execute.last_variants),
    }
    return result, counter, report


def _run_dense(e: TensorExpr, bindings, out_format, weights, timed: bool):
    """All-dense expressions: torch (cuBLAS, TF32 off), the paper's "dense -> torch" branch
    (`engine.py:687-701`). ``timed`` adds the device synchronisation for ``wall_time_ns``."""
    fmt = out_format if out_format is not None else dense_format(e.output_shape)
    sched = schedule(e, dense_format(e.output_shape), weights)
    ctx = _Ctx(sched, bindings, dense_format(e.output_shape), None)
    _require_device(ctx.tensor_of.values())
    t0 = time.perf_counter_ns()
    acc = None
    for term in e.terms():
        r = _dense_einsum(ctx, term, e.output_indices)
        acc = r if acc is None else acc + r
    if timed:
        torch.cuda.synchronize()
    wall = time.perf_counter_ns() - t0
    result = _dense_result(e.output_name, acc)
    if fmt.has_sparse_levels or fmt.mode_ordering != tuple(range(fmt.order)):
        from .tensor import from_dense

        result = from_dense(acc, fmt, name=e.output_name)
    report = {"path": "dense", "inferred_format": infer_format(e).name(), "schedule": None,
              "counters": None, "wall_time_ns": wall, "variants": ["dense:torch"]}
    return result, None, report


def _plan(e: TensorExpr, out_format, tile_size, tiling, weights):
    """(output format, tiled schedule), memoised on the expression: the plan depends only on
    the expression (whose operands are immutable and may only be rebound to tensors of the
    same shape and format) and the options."""
    plans = e.__dict__.setdefault("_plans", {})
    key = (out_format, tile_size, tiling, weights)
    got = plans.get(key)
    if got is None:
        out_fmt = out_format if out_format is not None else infer_format(e)
        sched = schedule(e, out_fmt, weights)
        if tiling:
            sched = tile(e, sched, tile_size)
        got = plans[key] = (out_fmt, sched)
    return got


def run(e: TensorExpr, bindings: dict | None = None, out_format: TensorFormat | None = None,
        tile_size: int = DEFAULT_TILE_SIZE, tiling: bool = True, weights: CostModel = CostModel(),
        variant: str | None = None) -> Tensor:
    """Plan + execute (`engine.py:721-724`). Asynchronous: the kernels are queued on the
    current CUDA stream and the call returns without waiting for them (reading the result
    on the host — ``to_dense``, ``nnz`` of a sparse result — synchronises)."""
    if bindings:
        for a in e.accesses:
            t = bindings.get(a.tensor.name)
            if t is not None and t.shape != a.tensor.shape:
                raise ShapeError(f"binding for {a.tensor.name} has shape {t.shape}")
    if all(not a.tensor.format.has_sparse_levels for a in e.accesses):
        return _run_dense(e, bindings, out_format, weights, timed=False)[0]
    _, sched = _plan(e, out_format, tile_size, tiling, weights)
    return execute(sched, bindings, variant=variant)[0]
