"""Exact ``OpCounter`` for expressions that run on the device loop-nest walker.

The reference counts work inside its interpreter (`/root/reference/pkg/src/sparsetc/engine.py:51-68`):
``scalar_mults`` / ``scalar_adds`` per scalar (or vectorised) multiply / add, and
``iterator_advances`` per cursor movement -- a ``bind`` of a compressed or coordinate
level (`engine.py:116-127, 158-165`), the scan of the smallest segment of an
intersection and the seeks of the others (`_intersect_sorted`, `engine.py:208-221`), the
merge of a union (`engine.py:224-230`), one step per tile block (`engine.py:358-365`),
each coordinate of a vectorised dense tail (`engine.py:413-431, 534-563`) and of a
full-range outer loop of a sparse output (`engine.py:609-611`). The kernels fill the
counters from closed forms; this module reproduces the interpreter's counting for any
other expression by walking the same loop nest breadth-first on the device: the frontier
of nodes advances one loop at a time (``generic._Cursor``: segment expansion, sorted-key
``find``), and each rule above becomes a sum over the frontier. Nothing is evaluated; only
the iteration space is enumerated, exactly as the reference visits it (the smallest
segment of every intersection is found per node, so its seek counts follow the
reference's order; union / full-range outer loops of sparse outputs track which terms
stay bound per node).
"""

from __future__ import annotations

import torch

from .expr import index_extents
from .generic import MAX_ROWS, TooLargeForGenericWalk, _Cursor
from .tiling import expanded_loops


def _arange(n, dev):
    return torch.arange(n, dtype=torch.long, device=dev)


class _Counts:
    def __init__(self):
        self.mults = 0
        self.adds = 0
        self.iters = 0


class _Front:
    """A frontier of loop-nest nodes for one term: per-row cursor states and tile blocks."""

    def __init__(self, n, cursors, blocks, dev):
        self.n = n                    # number of nodes
        self.cursors = cursors        # access id -> _Cursor (rows = nodes)
        self.blocks = blocks          # var -> block index per node
        self.dev = dev

    def take(self, rows: torch.Tensor) -> "_Front":
        cur = {}
        for k, c in self.cursors.items():
            c2 = c.clone()
            c2.take(rows)
            cur[k] = c2
        return _Front(int(rows.numel()), cur, {v: b[rows] for v, b in self.blocks.items()}, self.dev)

    @staticmethod
    def cat(parts: list, template: "_Front") -> "_Front":
        parts = [p for p in parts if p.n > 0]
        if not parts:
            return template.take(torch.zeros(0, dtype=torch.long, device=template.dev))
        cur = {k: _Cursor.cat([p.cursors[k] for p in parts]) for k in parts[0].cursors}
        blocks = {v: torch.cat([p.blocks[v] for p in parts]) for v in parts[0].blocks}
        return _Front(sum(p.n for p in parts), cur, blocks, parts[0].dev)


def _check(n):
    if n > MAX_ROWS:
        raise TooLargeForGenericWalk(f"loop nest frontier of {n} nodes")


class _TermCount:
    """One product term: its sparse accesses' cursor chains and dense readers."""

    def __init__(self, term, walk_of, dev):
        self.accesses = term
        self.vars = {v for a in term for v in a.indices}
        self.sparse = {}                  # access id -> (tensor, chain)
        for a in term:
            t = walk_of[id(a)]
            if t.format.has_sparse_levels:
                self.sparse[id(a)] = (t, tuple(a.indices[d] for d in t.format.mode_ordering))
        self.dev = dev

    def root(self) -> _Front:
        cur = {k: _Cursor(t, chain, self.dev) for k, (t, chain) in self.sparse.items()}
        return _Front(1, cur, {}, self.dev)

    def participants(self, front: _Front, var):
        """Cursor keys whose next unbound level stores ``var``, in access order."""
        out = []
        for a in self.accesses:
            c = front.cursors.get(id(a))
            if c is not None and c.depth < len(c.chain) and c.chain[c.depth] == var:
                out.append(id(a))
        return out


def _range(front: _Front, var, ext, tile):
    """(lo, length) per node of a loop over ``var``: its tile block's range or the full extent."""
    b = front.blocks.get(var)
    if b is None:
        return torch.zeros(front.n, dtype=torch.long, device=front.dev), torch.full(
            (front.n,), ext, dtype=torch.long, device=front.dev)
    lo = b * tile
    return lo, torch.clamp(ext - lo, max=tile)


def _expand_range(front: _Front, parts, var, ext, tile):
    """Children of a loop with no sparse participant (coordinates = the range)."""
    lo, ln = _range(front, var, ext, tile)
    total = int(ln.sum().item()) if front.n else 0
    _check(total)
    rows = torch.repeat_interleave(_arange(front.n, front.dev), ln)
    first = torch.cumsum(ln, 0) - ln
    coord = lo[rows] + (_arange(total, front.dev) - first[rows])
    child = front.take(rows)
    for k in parts:
        child.cursors[k].bind_dense(coord)
        child.cursors[k].depth += 1
    return child, coord


def _intersect(front: _Front, sparse_keys, dense_keys, cnt: _Counts):
    """Children of a loop whose coordinates are the intersection of the sparse participants'
    segments, with the reference's counting: the smallest segment (first minimum) is scanned,
    the others are seeked in list order while the running result is non-empty."""
    k = len(sparse_keys)
    lens = torch.stack([front.cursors[s].seg_len() for s in sparse_keys]) if front.n else torch.zeros(
        (k, 0), dtype=torch.long, device=front.dev)
    base = torch.argmin(lens, dim=0) if front.n else torch.zeros(0, dtype=torch.long, device=front.dev)
    cnt.iters += int(lens.gather(0, base[None, :]).sum().item()) if front.n else 0
    groups, coords = [], []
    for b in range(k):
        rows_b = torch.nonzero(base == b).flatten()
        if rows_b.numel() == 0:
            continue
        sub = front.take(rows_b)
        bk = sparse_keys[b]
        prow, coord = sub.cursors[bk].expand()
        _check(int(prow.numel()))
        for key, c in sub.cursors.items():
            if key != bk:
                c.take(prow)
        for key in sub.blocks:
            sub.blocks[key] = sub.blocks[key][prow]
        alive = torch.ones(prow.numel(), dtype=torch.bool, device=front.dev)
        prev = lens[b, rows_b]
        for o in sparse_keys:
            if o == bk:
                continue
            ok = sub.cursors[o].find(coord)
            alive &= ok
            now = torch.bincount(prow[alive], minlength=rows_b.numel())
            cnt.iters += int(((now + 1) * (prev > 0)).sum().item())
            prev = now
        sel = torch.nonzero(alive).flatten()
        sub.n = int(sel.numel())
        for c in sub.cursors.values():
            c.take(sel)
        for key in sub.blocks:
            sub.blocks[key] = sub.blocks[key][sel]
        coord = coord[sel]
        for key in sparse_keys + dense_keys:
            if key in dense_keys:
                sub.cursors[key].bind_dense(coord)
            sub.cursors[key].depth += 1
        groups.append(sub)
        coords.append(coord)
    child = _Front.cat(groups, front)
    if not groups:
        for key in sparse_keys + dense_keys:
            child.cursors[key].depth += 1
    coord = torch.cat(coords) if coords else torch.zeros(0, dtype=torch.long, device=front.dev)
    cnt.iters += k * child.n  # one bind per sparse participant per coordinate
    return child, coord


def _step(ts: _TermCount, front: _Front, var, ext, tile, cnt: _Counts):
    parts = ts.participants(front, var)
    sparse = [p for p in parts if front.cursors[p].next_is_sparse()]
    dense = [p for p in parts if p not in sparse]
    if sparse:
        return _intersect(front, sparse, dense, cnt)[0]
    return _expand_range(front, parts, var, ext, tile)[0]


def _blocks(front: _Front, var, ext, tile, cnt: _Counts) -> _Front:
    nb = -(-ext // tile)
    cnt.iters += front.n * nb
    _check(front.n * nb)
    rows = _arange(front.n, front.dev).repeat_interleave(nb)
    child = front.take(rows)
    child.blocks[var] = _arange(nb, front.dev).repeat(front.n)
    return child


def _count_term(ts: _TermCount, front: _Front, steps, keys, sink, ext, tile, cnt: _Counts, exclude=frozenset()):
    """``_run_term`` (engine.py:365-483) counted over a frontier of start nodes. ``sink`` is
    "scalar" (one add per key: the dense output's and the workspace's accumulate) or a tuple
    ("vector", tail var, number of consumed tail accesses) for the vectorised dense tail."""
    binding_depth = {s.var: i for i, s in enumerate(steps) if s.role != "block"}
    consumed_at = {i: [] for i in range(len(steps))}
    n_pre = 0
    for a in ts.accesses:
        if id(a) in exclude:
            continue
        depths = [binding_depth[v] for v in a.indices if v in binding_depth]
        if depths:
            consumed_at[max(depths)].append(a)
        else:
            n_pre += 1
    key_depths = [binding_depth[v] for v in keys if v in binding_depth]
    kd = max(key_depths) if key_depths else -1
    cnt.mults += front.n * max(n_pre - 1, 0)
    carry_none = n_pre == 0
    for d in range(kd + 1):
        st = steps[d]
        if st.role == "block":
            front = _blocks(front, st.var, ext[st.var], tile, cnt)
            continue
        front = _step(ts, front, st.var, ext[st.var], tile, cnt)
        c = len(consumed_at[d])
        if c:
            cnt.mults += front.n * (c - 1 if carry_none else c)
            carry_none = False
    # emit: the reduction below the deepest key, the carry times its total, the sink
    if kd + 1 < len(steps):
        _count_reduce(ts, front, steps, kd + 1, consumed_at, ext, tile, cnt)
        if not carry_none:
            cnt.mults += front.n
        carry_none = False
    if sink == "scalar":
        cnt.adds += front.n
        return
    _, tail_var, n_tail = sink
    _, ln = _range(front, tail_var, ext[tail_var], tile)
    tot = int(ln.sum().item()) if front.n else 0
    cnt.mults += tot * max(n_tail - 1, 0)
    if n_tail and not carry_none:
        cnt.mults += tot
    cnt.iters += tot
    cnt.adds += tot


def _count_reduce(ts, front, steps, d, consumed_at, ext, tile, cnt):
    """``reduce_zone`` (engine.py:404-442) over every node of ``front``."""
    if front.n == 0:
        return
    st = steps[d]
    if st.role == "block":
        _count_reduce(ts, _blocks(front, st.var, ext[st.var], tile, cnt), steps, d + 1, consumed_at, ext, tile, cnt)
        return
    parts = ts.participants(front, st.var)
    c = len(consumed_at[d])
    if d == len(steps) - 1 and not parts and c and all(id(a) not in ts.sparse for a in consumed_at[d]):
        # vectorised innermost dense reduction: products, one advance and one add per coordinate
        _, ln = _range(front, st.var, ext[st.var], tile)
        tot = int(ln.sum().item())
        cnt.mults += tot * (c - 1)
        cnt.iters += tot
        cnt.adds += tot
        return
    child = _step(ts, front, st.var, ext[st.var], tile, cnt)
    cnt.mults += child.n * max(c - 1, 0)
    if d + 1 < len(steps):
        _count_reduce(ts, child, steps, d + 1, consumed_at, ext, tile, cnt)
        if c:
            cnt.mults += child.n
    cnt.adds += child.n


def count_ops(sched, walk_of: dict, out_fmt):
    """(scalar_mults, scalar_adds, iterator_advances) of the reference interpreter for
    ``sched`` over the (storage-order-converted) operands ``walk_of``, into ``out_fmt``."""
    e = sched.expr
    ext = index_extents(e)
    tile = sched.tile_size or 1
    steps = expanded_loops(sched)
    dev = next(iter(walk_of.values())).storage.values.device
    out_vars = e.output_indices
    out_chain = tuple(out_vars[d] for d in out_fmt.mode_ordering)
    terms = [_TermCount(t, walk_of, dev) for t in e.terms()]
    cnt = _Counts()
    if not out_fmt.has_sparse_levels:
        for ts in terms:
            st = [s for s in steps if s.var in ts.vars or s.var in out_vars]
            binding = [s for s in st if s.role != "block"]
            fast = bool(st) and st[-1].role != "block" and st[-1].var in out_vars and bool(binding) and \
                binding[-1] is st[-1]
            tail = []
            if fast:
                tail = [a for a in ts.accesses if st[-1].var in a.indices]
                fast = all(id(a) not in ts.sparse for a in tail)
            if not fast:
                _count_term(ts, ts.root(), st, tuple(out_vars), "scalar", ext, tile, cnt)
                continue
            head = st[:-1]
            head_keys = tuple(s.var for s in binding[:-1])
            _count_term(ts, ts.root(), head, head_keys, ("vector", st[-1].var, len(tail)), ext, tile, cnt,
                        exclude=frozenset(id(a) for a in tail))
        return cnt.mults, cnt.adds, cnt.iters
    _count_sparse_output(terms, steps, out_chain, ext, tile, cnt, dev)
    return cnt.mults, cnt.adds, cnt.iters


def _count_sparse_output(terms, steps, out_chain, ext, tile, cnt, dev):
    """``_run_sparse_output`` (engine.py:577-644): leading full loops over output indices
    iterate the union of the terms' intersections (or the full range when a term has no
    sparse participant), each term stays bound where its cursors hold the coordinate; then
    every bound term runs its inner nest into the workspace (one add per key)."""
    n_outer = 0
    for s, v in zip(steps, out_chain):
        if s.role == "full" and s.var == v:
            n_outer += 1
        else:
            break
    outer, inner = steps[:n_outer], steps[n_outer:]
    keys = out_chain[n_outer:]
    fronts = [ts.root() for ts in terms]             # per term: its nodes (rows of the shared frontier)
    node_of = [torch.zeros(1, dtype=torch.long, device=dev) for _ in terms]  # shared node id per term row
    n_nodes = 1
    for st in outer:
        var, e_v = st.var, ext[st.var]
        # per node: does some active term iterate the full range (no sparse participant)?
        full = torch.zeros(n_nodes, dtype=torch.bool, device=dev)
        streams = []   # (term index, child front, coords, parent node ids)
        for i, ts in enumerate(terms):
            f = fronts[i]
            if f.n == 0:
                continue
            parts = ts.participants(f, var) if var in ts.vars else []
            sparse = [p for p in parts if f.cursors[p].next_is_sparse()]
            if not sparse:
                full[node_of[i]] = True
                continue
            sub = _Counts()
            lens = torch.stack([f.cursors[s].seg_len() for s in sparse])
            # the stream is the term's intersection (counted as the reference counts it)
            child, coord = _intersect_stream(f, sparse, lens, sub)
            cnt.iters += sub.iters
            streams.append((i, child, coord))
        # coordinates per node: full range, else the union of the streams
        full_nodes = torch.nonzero(full).flatten()
        cnt.iters += int(full_nodes.numel()) * e_v
        union_keys = []
        for i, child, coord in streams:
            pn = node_of[i][child.parent]
            keep = ~full[pn]
            cnt.iters += int(keep.sum().item())                   # union: each stream scanned once
            union_keys.append(pn[keep] * e_v + coord[keep])
        full_keys = (full_nodes[:, None] * e_v + _arange(e_v, dev)[None, :]).flatten()
        all_keys = torch.unique(torch.cat(union_keys + [full_keys])) if (union_keys or full_keys.numel()) else \
            torch.zeros(0, dtype=torch.long, device=dev)
        _check(int(all_keys.numel()))
        new_nodes = int(all_keys.numel())
        # bind every term at every child coordinate of its nodes (attempt counts until a failure)
        for i, ts in enumerate(terms):
            f = fronts[i]
            if f.n == 0:
                continue
            parts = ts.participants(f, var) if var in ts.vars else []
            # children of this term's nodes: every key of its node
            lo = torch.searchsorted(all_keys, node_of[i] * e_v)
            hi = torch.searchsorted(all_keys, node_of[i] * e_v + e_v)
            ln = hi - lo
            rows = torch.repeat_interleave(_arange(f.n, dev), ln)
            first = torch.cumsum(ln, 0) - ln
            kidx = lo[rows] + (_arange(int(rows.numel()), dev) - first[rows])
            coord = all_keys[kidx] % e_v
            child = f.take(rows)
            ok = torch.ones(child.n, dtype=torch.bool, device=dev)
            for p in parts:
                c = child.cursors[p]
                if c.next_is_sparse():
                    cnt.iters += int(ok.sum().item())        # a bind attempt on every still-bound child
                    ok &= c.find(coord)
                else:
                    c.bind_dense(coord)
                c.depth += 1
            sel = torch.nonzero(ok).flatten()
            fronts[i] = child.take(sel)
            node_of[i] = kidx[sel]
        n_nodes = new_nodes
    term_inner = [[s for s in inner if s.var in ts.vars or s.var in keys] for ts in terms]
    for i, ts in enumerate(terms):
        if fronts[i].n:
            _count_term(ts, fronts[i], term_inner[i], tuple(keys), "scalar", ext, tile, cnt)


def _intersect_stream(front: _Front, sparse_keys, lens, cnt: _Counts):
    """The term's intersection over its sparse participants for every node (children carry
    ``parent`` = node row), counted like ``_intersect_sorted``; no bind counts (those come with
    the union's per-term bind attempts)."""
    k = len(sparse_keys)
    base = torch.argmin(lens, dim=0)
    cnt.iters += int(lens.gather(0, base[None, :]).sum().item())
    parents, coords = [], []
    for b in range(k):
        rows_b = torch.nonzero(base == b).flatten()
        if rows_b.numel() == 0:
            continue
        sub = front.take(rows_b)
        bk = sparse_keys[b]
        prow, coord = sub.cursors[bk].clone().expand()
        alive = torch.ones(prow.numel(), dtype=torch.bool, device=front.dev)
        prev = lens[b, rows_b]
        for o in sparse_keys:
            if o == bk:
                continue
            c = sub.cursors[o].clone()
            c.take(prow)
            alive &= c.find(coord)
            now = torch.bincount(prow[alive], minlength=rows_b.numel())
            cnt.iters += int(((now + 1) * (prev > 0)).sum().item())
            prev = now
        parents.append(rows_b[prow[alive]])
        coords.append(coord[alive])
    child = _Front(0, {}, {}, front.dev)
    child.parent = torch.cat(parents) if parents else torch.zeros(0, dtype=torch.long, device=front.dev)
    coord = torch.cat(coords) if coords else torch.zeros(0, dtype=torch.long, device=front.dev)
    return child, coord
