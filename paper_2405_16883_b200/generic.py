"""Device loop-nest walker for expressions that have no dedicated kernel.

The reference runs every expression through one interpreter (`engine.py:365-483`
`_run_term`, `engine.py:487-573` dense output, `engine.py:577-644` sparse output):
loops in schedule order, each loop iterating the intersection of the segments of
the sparse operands whose next storage level it binds (`_step_coords`,
`engine.py:327-336`; `_intersect_sorted`, `engine.py:208-221`) or the full extent
when none does; a sparse output stores every key the nest visits, reductions that
come out empty included (`emit`, `engine.py:453-460`).

The hot path (SpMM / SDDMM / MTTKRP / SpGEMM / CSR element-wise) has its own
kernels; this module covers everything else *on the device*, breadth-first: the
whole frontier of partial loop bindings advances one loop at a time as torch
device tensors (one row per binding, with the cursor position of every sparse
operand), so the iteration space is exactly the reference's:

* a loop whose sparse participants exist expands each row by its first
  participant's segment (compressed level: ``crd[pos[p]:pos[p+1]]``; coordinate
  level: the distinct values of the bound run) and keeps the coordinates the other
  participants hold (a sorted-key ``searchsorted`` per level, the vectorised
  ``bind``); dense-level participants only advance their position;
* a loop with no sparse participant expands by its full extent;
* the keys a term visits are snapshotted after its deepest output loop, so a key
  whose inner reduction is empty is still stored (value 0.0), as in the reference;
* products and sums run in float64 on the device — per-key sums by a stable sort and a
  segmented reduction, no atomics, so results are bit-reproducible — the result is
  rounded once to float32 (storage dtype), and the output is assembled by ``tensor._assemble_sorted``
  (the device restatement of `_assemble_presorted`, `tensor.py:162-219`).

Operands stored in an order that violates the loop order are converted first
(`engine.py:313-318`). Tiling is bit-neutral in the reference
(`tests/test_acceptance.py:85-98`) and does not change the walk. The OpCounter of this
path is the interpreter's exact count, from a second breadth-first enumeration of the
reference's own loop nest (tile blocks, intersection order, vectorised tails and all:
``walk_count.count_ops``), pinned to the reference's counters on every fixture.
"""

from __future__ import annotations

import math

import torch

from .expr import TensorExpr, index_extents
from .formats import LevelFormat, TensorFormat
from .scheduler import Schedule, _desired_ordering, _violates
from .tensor import DenseLevel, Tensor, TensorStorage, VALUE_DTYPE, _assemble_sorted, convert

# Frontier rows above which the walk refuses (memory: ~8 bytes x (vars + cursors) per row).
MAX_ROWS = 1 << 27


class TooLargeForGenericWalk(RuntimeError):
    pass


def _check_rows(counts: torch.Tensor) -> None:
    total = int(counts.sum().item()) if counts.numel() else 0
    if total > MAX_ROWS:
        raise TooLargeForGenericWalk(f"loop nest frontier of {total} rows")


def _arange(n, dev):
    return torch.arange(n, dtype=torch.long, device=dev)


class _Cursor:
    """One sparse operand's position in its level structure, per frontier row."""

    def __init__(self, t: Tensor, chain: tuple, dev):
        self.t = t
        self.chain = chain
        self.depth = 0
        fmt = t.format
        self.coo = fmt.is_coordinate
        self.kinds = fmt.levels
        self.extents = [fmt.level_extent(k) for k in range(fmt.order)]
        self.values = t.storage.values
        self.dev = dev
        n = int(self.values.numel())
        if self.coo:
            self.crds = [lv.crd.to(torch.long) for lv in t.storage.levels]
            self.lo = torch.zeros(1, dtype=torch.long, device=dev)
            self.hi = torch.full((1,), n, dtype=torch.long, device=dev)
        else:
            self.p = torch.zeros(1, dtype=torch.long, device=dev)
        self._keys = {}

    def next_var(self):
        return self.chain[self.depth] if self.depth < len(self.chain) else None

    def next_is_sparse(self) -> bool:
        return self.coo or self.kinds[self.depth] is not LevelFormat.DENSE

    def take(self, rows: torch.Tensor) -> None:
        if self.coo:
            self.lo, self.hi = self.lo[rows], self.hi[rows]
        else:
            self.p = self.p[rows]

    def clone(self) -> "_Cursor":
        c = object.__new__(_Cursor)
        c.__dict__.update(self.__dict__)
        return c

    @staticmethod
    def cat(parts: list) -> "_Cursor":
        """Row-wise concatenation of clones of one cursor (same depth)."""
        c = parts[0].clone()
        if c.coo:
            c.lo = torch.cat([x.lo for x in parts])
            c.hi = torch.cat([x.hi for x in parts])
        else:
            c.p = torch.cat([x.p for x in parts])
        return c

    def seg_len(self) -> torch.Tensor:
        """Per row, the number of coordinates the next (sparse) level iterates: the segment
        length of a compressed level, the distinct values of the bound run of a coordinate level
        (the reference's ``segment_coords``, engine.py:111-114, 150-152)."""
        if self.coo:
            rows, _ = self.clone().expand()
            return torch.bincount(rows, minlength=self.lo.numel())
        pos = self.t.storage.levels[self.depth].pos.to(torch.long)
        return pos[self.p + 1] - pos[self.p]

    # -- sorted search keys per level (parent id * extent + coordinate) --------------
    def _level_key(self, d: int) -> torch.Tensor:
        if d not in self._keys:
            ext = self.extents[d]
            if self.coo:
                n = self.crds[0].numel()
                gid = torch.zeros(n, dtype=torch.long, device=self.dev)
                if d > 0 and n > 1:
                    change = torch.zeros(n, dtype=torch.bool, device=self.dev)
                    for k in range(d):
                        change[1:] |= self.crds[k][1:] != self.crds[k][:-1]
                    gid = torch.cumsum(change.to(torch.long), 0)
                self._keys[d] = (gid, gid * ext + self.crds[d])
            else:
                lv = self.t.storage.levels[d]
                pos = lv.pos.to(torch.long)
                parent = torch.repeat_interleave(_arange(pos.numel() - 1, self.dev), pos[1:] - pos[:-1])
                self._keys[d] = (parent, parent * ext + lv.crd.to(torch.long))
        return self._keys[d]

    # -- expansion by this cursor's own segment ------------------------------------
    def expand(self):
        """Rows x segment: returns (row index, coordinate) per candidate and moves self."""
        d = self.depth
        if self.coo:
            lo, hi = self.lo, self.hi
            counts = hi - lo
            _check_rows(counts)
            rows = torch.repeat_interleave(_arange(lo.numel(), self.dev), counts)
            first = torch.cumsum(counts, 0) - counts
            ent = lo[rows] + (_arange(rows.numel(), self.dev) - first[rows])
            col = self.crds[d]
            keep = torch.ones(ent.numel(), dtype=torch.bool, device=self.dev)
            if ent.numel():
                keep = (ent == lo[rows]) | (col[ent] != col[(ent - 1).clamp(min=0)])
            rows, ent = rows[keep], ent[keep]
            # a distinct value's run ends where the next kept entry of the same row starts
            nxt = torch.empty_like(ent)
            if ent.numel():
                nxt[:-1] = ent[1:]
                nxt[-1] = hi[rows[-1]]
                last = torch.ones(ent.numel(), dtype=torch.bool, device=self.dev)
                last[:-1] = rows[1:] != rows[:-1]
                nxt = torch.where(last, hi[rows], nxt)
            self.lo, self.hi = ent, nxt
            return rows, col[ent]
        lv = self.t.storage.levels[d]
        pos = lv.pos.to(torch.long)
        lo, hi = pos[self.p], pos[self.p + 1]
        counts = hi - lo
        _check_rows(counts)
        rows = torch.repeat_interleave(_arange(lo.numel(), self.dev), counts)
        first = torch.cumsum(counts, 0) - counts
        ent = lo[rows] + (_arange(rows.numel(), self.dev) - first[rows])
        self.p = ent
        return rows, lv.crd.to(torch.long)[ent]

    # -- bind a coordinate found elsewhere (intersection) --------------------------
    def find(self, coord: torch.Tensor) -> torch.Tensor:
        """Move to ``coord`` in each row's segment; returns the rows that hold it."""
        d = self.depth
        ext = self.extents[d]
        gid, key = self._level_key(d)
        if self.coo:
            q = gid[self.lo.clamp(max=max(gid.numel() - 1, 0))] * ext + coord if gid.numel() else coord
            left = torch.searchsorted(key, q, right=False)
            right = torch.searchsorted(key, q, right=True)
            ok = (right > left) & (self.hi > self.lo)
            self.lo, self.hi = left, right
            return ok
        q = self.p * ext + coord
        idx = torch.searchsorted(key, q)
        ok = idx < key.numel()
        ok &= key[idx.clamp(max=max(key.numel() - 1, 0))] == q if key.numel() else torch.zeros_like(ok)
        self.p = idx
        return ok

    def bind_dense(self, coord: torch.Tensor) -> None:
        self.p = self.p * self.extents[self.depth] + coord

    def value(self) -> torch.Tensor:
        v = self.values.to(torch.float64)
        return v[self.lo] if self.coo else v[self.p]


def _dense_strides(t: Tensor) -> list:
    fmt = t.format
    strides = [0] * fmt.order
    acc = 1
    for k in reversed(range(fmt.order)):
        strides[fmt.mode_ordering[k]] = acc
        acc *= fmt.level_extent(k)
    return strides


def _walk_term(term, tensor_of, loop_order, out_chain, ext, dev):
    """Returns (visited keys as linear out-chain offsets (unique, sorted), key of each
    final row, product of each final row) for one product term."""
    term_vars = {v for a in term for v in a.indices}
    steps = [v for v in loop_order if v in term_vars or v in out_chain]
    out_set = set(out_chain)
    last_out = max((i for i, v in enumerate(steps) if v in out_set), default=-1)
    cursors, readers = [], []
    for a in term:
        t = tensor_of[id(a)]
        if t.format.has_sparse_levels:
            cursors.append((a, _Cursor(t, tuple(a.indices[d] for d in t.format.mode_ordering), dev)))
        else:
            readers.append((a, t))
    n_rows = 1
    coords: dict = {}
    out_strides, acc = {}, 1
    for v in reversed(out_chain):
        out_strides[v] = acc
        acc *= ext[v]
    if acc >= 2**62:
        raise TooLargeForGenericWalk("output index space exceeds 2^62 positions")

    def lin_of(rows_coords):
        lin = torch.zeros(n_rows, dtype=torch.long, device=dev)
        for v in out_chain:
            lin += rows_coords[v] * out_strides[v]
        return lin

    keys = torch.zeros(1, dtype=torch.long, device=dev) if last_out < 0 else None
    for si, v in enumerate(steps):
        parts = [c for _, c in cursors if c.next_var() == v]
        sparse = [c for c in parts if c.next_is_sparse()]
        if sparse:
            base = sparse[0]
            others = [c for c in parts if c is not base]
            # cursors not moved by this loop keep their state per row
            idle = [c for _, c in cursors if c not in parts]
            rows, coord = base.expand()
            for c in others + idle:
                c.take(rows)
            keep = None
            for c in others:
                if c.next_is_sparse():
                    ok = c.find(coord)
                    keep = ok if keep is None else keep & ok
            if keep is not None:
                sel = torch.nonzero(keep).flatten()
                rows, coord = rows[sel], coord[sel]
                for c in parts + idle:
                    c.take(sel)
            for c in others:
                if not c.next_is_sparse():
                    c.bind_dense(coord)
        else:
            e = ext[v]
            total = n_rows * e
            if total > MAX_ROWS:
                raise TooLargeForGenericWalk(f"loop nest frontier of {total} rows")
            rows = _arange(n_rows, dev).repeat_interleave(e)
            coord = _arange(e, dev).repeat(n_rows)
            for _, c in cursors:
                c.take(rows)
            for c in parts:
                c.bind_dense(coord)
        for c in parts:
            c.depth += 1
        coords = {u: x[rows] for u, x in coords.items()}
        coords[v] = coord
        n_rows = int(coord.numel())
        if n_rows > MAX_ROWS:
            raise TooLargeForGenericWalk(f"loop nest frontier of {n_rows} rows")
        if si == last_out:
            keys = torch.unique(lin_of(coords))
    # product of every factor at each full binding (float64)
    prod = torch.ones(n_rows, dtype=torch.float64, device=dev)
    for a, c in cursors:
        prod = prod * c.value()
    for a, t in readers:
        strides = _dense_strides(t)
        off = torch.zeros(n_rows, dtype=torch.long, device=dev)
        for d, u in enumerate(a.indices):
            off += coords[u] * strides[d]
        prod = prod * t.storage.values.to(torch.float64)[off]
    row_key = lin_of(coords) if out_chain else torch.zeros(n_rows, dtype=torch.long, device=dev)
    return keys, row_key, prod


def execute_generic(sched: Schedule, tensor_of: dict, out_fmt: TensorFormat, counter) -> Tensor:
    """Evaluate ``sched.expr`` into ``out_fmt`` by the breadth-first device walk."""
    e: TensorExpr = sched.expr
    ext = index_extents(e)
    order = tuple(sched.loop_order)
    pos = {v: i for i, v in enumerate(order)}
    dev = next(iter(tensor_of.values())).storage.values.device
    # operands whose storage order violates the loop order are re-stored first
    walk_of, conv = {}, {}
    for a in e.accesses:
        t = tensor_of[id(a)]
        chain = tuple(a.indices[d] for d in t.format.mode_ordering)
        if t.format.has_sparse_levels and _violates(pos, chain):
            target = _desired_ordering(a, pos)
            key = (id(t), target)
            if key not in conv:
                conv[key] = convert(t, t.format.with_mode_ordering(target))
            t = conv[key]
        walk_of[id(a)] = t
    out_vars = e.output_indices
    out_chain = tuple(out_vars[d] for d in out_fmt.mode_ordering)
    shape = tuple(ext[v] for v in out_vars)
    # the reference interpreter's exact counters: its loop nest enumerated on the device
    from .walk_count import count_ops

    counter.add(*count_ops(sched, walk_of, out_fmt))
    all_keys, all_rows, all_prod = [], [], []
    for term in e.terms():
        keys, row_key, prod = _walk_term(term, walk_of, order, out_chain, ext, dev)
        all_keys.append(keys)
        all_rows.append(row_key)
        all_prod.append(prod)
    size = math.prod(ext[v] for v in out_chain)
    # per-key sums in a fixed order (stable sort by key, terms in expression order, then a
    # segmented reduction): no floating-point atomics, bit-reproducible run to run
    ukeys, sums = _segment_sums(torch.cat(all_rows), torch.cat(all_prod))
    if not out_fmt.has_sparse_levels:
        flat = torch.zeros(size, dtype=torch.float64, device=dev)
        flat[ukeys] = sums
        st = TensorStorage(out_fmt, tuple(DenseLevel(out_fmt.level_extent(k)) for k in range(out_fmt.order)),
                           flat.to(VALUE_DTYPE))
        st.validate()
        return Tensor(e.output_name, shape, st)
    keys = torch.unique(torch.cat(all_keys))
    vals = torch.zeros(keys.numel(), dtype=torch.float64, device=dev)
    if ukeys.numel():
        vals[torch.searchsorted(keys, ukeys)] = sums
    perm_cols = torch.empty((keys.numel(), len(out_chain)), dtype=torch.long, device=dev)
    rem = keys.clone()
    for k in reversed(range(len(out_chain))):
        e_k = ext[out_chain[k]]
        perm_cols[:, k] = rem % e_k
        rem = rem // e_k
    return _assemble_sorted(shape, out_fmt, perm_cols, vals.to(VALUE_DTYPE), e.output_name)


def _segment_sums(row_key: torch.Tensor, prod: torch.Tensor):
    """(distinct keys ascending, float64 sum of each key's products in input order)."""
    if not row_key.numel():
        return row_key, prod
    order = torch.argsort(row_key, stable=True)
    sk, sv = row_key[order], prod[order]
    ukeys, counts = torch.unique_consecutive(sk, return_counts=True)
    return ukeys, torch.segment_reduce(sv, "sum", lengths=counts)
