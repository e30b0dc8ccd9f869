"""Vectorised float64 restatements of the reference engine — TEST ONLY.

Each function names the reference code whose arithmetic order it reproduces.
Inputs are numpy arrays (int64/int32 indices, float64 values); the same
fp32-rounded values given to the GPU are upcast to float64 here.
"""

from __future__ import annotations

import numpy as np


def _row_lengths(rowptr):
    return np.diff(np.asarray(rowptr, dtype=np.int64))


def spmm_csr(rowptr, colidx, vals, B, addend=None):
    """C = A @ B (+ addend) for CSR A, dense B.

    Reference: `_run_dense_output` + `vector_sink` (engine.py:487-565): the
    output starts at 0.0 and for every stored a_ij, in ascending j, adds
    ``a_ij * B[j, block]`` (engine.py:551-560). Column blocks (tiling.py:69-92)
    do not change any element's order. Position-major: step p folds the p-th
    entry of every row that has one, so each element's sum order is exact.
    A second additive term ``+ D(i,k)`` is added after the product term
    (terms run sequentially, engine.py:501).
    """
    rowptr = np.asarray(rowptr, dtype=np.int64)
    colidx = np.asarray(colidx, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    m = len(rowptr) - 1
    C = np.zeros((m, B.shape[1]), dtype=np.float64)
    lens = _row_lengths(rowptr)
    maxlen = int(lens.max()) if m else 0
    starts = rowptr[:-1]
    for p in range(maxlen):
        rows = np.flatnonzero(lens > p)
        pos = starts[rows] + p
        C[rows] += vals[pos][:, None] * B[colidx[pos]]
    if addend is not None:
        C += np.asarray(addend, dtype=np.float64)
    return C


def spmm_abs(rowptr, colidx, vals, B):
    """|A| @ |B|: the per-element magnitude bound used by the parity gate."""
    return spmm_csr(rowptr, colidx, np.abs(vals), np.abs(B))


def sddmm_csr(rowptr, colidx, maskvals, Q, K, tile: int | None = 64):
    """S[p] = m_ij * <q_i, k_j> for the stored (i, j) of the mask.

    Reference: `_run_sparse_output` -> `emit` -> `reduce_zone` (engine.py:404-461):
    the d loop is split into blocks of ``tile`` (tiling.py:81-90), each block is
    a vectorised product followed by a plain left-to-right sum from 0.0
    (engine.py:419-431), blocks are summed left to right from 0.0
    (engine.py:406-410), and the mask value multiplies the total last
    (engine.py:456-458). ``tile=None`` is the untiled plan (one sequential sum).
    """
    rowptr = np.asarray(rowptr, dtype=np.int64)
    colidx = np.asarray(colidx, dtype=np.int64)
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    m = len(rowptr) - 1
    rows = np.repeat(np.arange(m), _row_lengths(rowptr))
    prod = Q[rows] * K[colidx]  # (nnz, d): elementwise products, exact per element
    d = Q.shape[1]
    bounds = [(0, d)] if tile is None else [(lo, min(lo + tile, d)) for lo in range(0, d, tile)]
    total = np.zeros(len(colidx), dtype=np.float64)
    for lo, hi in bounds:
        part = np.zeros(len(colidx), dtype=np.float64)
        for x in range(lo, hi):
            part = part + prod[:, x]
        total = total + part
    mv = np.ones(len(colidx)) if maskvals is None else np.asarray(maskvals, dtype=np.float64)
    return mv * total


def sddmm_abs(rowptr, colidx, maskvals, Q, K):
    mv = None if maskvals is None else np.abs(maskvals)
    return sddmm_csr(rowptr, colidx, mv, np.abs(Q), np.abs(K))


def segment_softmax(rowptr, vals):
    """Row-wise softmax over each row's stored values (no reference symbol:
    the grammar has only + and *). exp(s - max) / sum."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    m = len(rowptr) - 1
    out = np.empty_like(vals)
    lens = _row_lengths(rowptr)
    rows = np.repeat(np.arange(m), lens)
    if len(vals) == 0:
        return out
    mx = np.full(m, -np.inf)
    np.maximum.at(mx, rows, vals)
    e = np.exp(vals - mx[rows])
    s = np.zeros(m)
    np.add.at(s, rows, e)
    out[:] = e / s[rows]
    return out


def sparse_attention(rowptr, colidx, maskvals, Q, K, V, scale):
    """O = softmax_rows(scale * SDDMM(Q, K; mask)) @ V, float64, unfused."""
    S = scale * sddmm_csr(rowptr, colidx, maskvals, Q, K)
    P = segment_softmax(rowptr, S)
    O = spmm_csr(rowptr, colidx, P, V)
    return S, P, O


def coo_segments(rows):
    """Distinct rows of a sorted COO row column and their entry offsets
    (the compressed i-level built by `_SparseOutputBuilder`, engine.py:233-253)."""
    rows = np.asarray(rows, dtype=np.int64)
    if len(rows) == 0:
        return np.zeros(0, np.int64), np.zeros(1, np.int64)
    first = np.ones(len(rows), dtype=bool)
    first[1:] = rows[1:] != rows[:-1]
    starts = np.flatnonzero(first)
    return rows[starts], np.append(starts, len(rows))


def spmm_coo(rows, cols, vals, B):
    """COO SpMM -> ([compressed, dense] i-crd, values (n_seg, K)).

    Reference: `_run_sparse_output` with the (i, k) Workspace (engine.py:577-608,
    71-90): every (i, k) accumulates ``a_ij * B[j, k]`` from 0.0 in ascending j,
    drained in key order -> the i-level holds the distinct rows.
    """
    seg_rows, seg_ptr = coo_segments(rows)
    C = spmm_csr(seg_ptr, cols, vals, B)
    return seg_rows, C


def mttkrp_coo(i, j, k, vals, B, C, b_first: bool = True):
    """M[i, r] = sum over stored (i,j,k) of (t * B[j,r]) * C[k,r] (B listed before C).

    Reference: `_run_sparse_output` with one Workspace keyed (i, r)
    (engine.py:577-608, 81-83); the fold order is term order at the deepest
    binding loop (engine.py:374-402): t at k, then B and C at r. Entries
    accumulate from 0.0 in the lexicographic (i, j, k) order.
    """
    seg_rows, seg_ptr = coo_segments(i)
    j = np.asarray(j, dtype=np.int64)
    k = np.asarray(k, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    n_seg = len(seg_rows)
    M = np.zeros((n_seg, B.shape[1]))
    lens = np.diff(seg_ptr)
    maxlen = int(lens.max()) if n_seg else 0
    starts = seg_ptr[:-1]
    for p in range(maxlen):
        segs = np.flatnonzero(lens > p)
        pos = starts[segs] + p
        t = vals[pos][:, None]
        if b_first:
            term = (t * B[j[pos]]) * C[k[pos]]
        else:
            term = (t * C[k[pos]]) * B[j[pos]]
        M[segs] += term
    return seg_rows, M


def mttkrp_abs(i, j, k, vals, B, C):
    return mttkrp_coo(i, j, k, np.abs(vals), np.abs(B), np.abs(C))


def spgemm_csr(ap, aj, av, bp, bj, bv):
    """C = A @ B for CSR A, CSR B -> CSR (rowptr, colidx, vals).

    Reference: `_run_sparse_output` with the [i, j, k] plan and a Workspace over
    k (engine.py:577-644, 71-90): for each row i, j ascending over A's row, k
    ascending over B's row j, ``ws[k] = ws.get(k, 0.0) + a_ij * b_jk``; the
    drain emits every touched k in order, zeros included. Vectorised as an
    expansion in (i, j, k) order, a stable sort by (i, k), and run sums from
    0.0 (``np.add.reduceat`` would pair-sum, so runs are folded position-major).
    """
    ap, aj, bp, bj = (np.asarray(x, dtype=np.int64) for x in (ap, aj, bp, bj))
    av, bv = np.asarray(av, dtype=np.float64), np.asarray(bv, dtype=np.float64)
    m = len(ap) - 1
    a_rows = np.repeat(np.arange(m), np.diff(ap))
    blen = np.diff(bp)[aj]
    # expand: product t belongs to A entry e = rep[t], B position bp[aj[e]] + offset
    rep = np.repeat(np.arange(len(aj)), blen)
    first = np.repeat(np.cumsum(blen) - blen, blen)
    bpos = bp[aj][rep] + (np.arange(len(rep)) - first)
    rows = a_rows[rep]
    keys = bj[bpos]
    prod = av[rep] * bv[bpos]
    order = np.lexsort((keys, rows))  # stable: equal (i, k) keep ascending j
    rows, keys, prod = rows[order], keys[order], prod[order]
    newrun = np.ones(len(keys), dtype=bool)
    newrun[1:] = (rows[1:] != rows[:-1]) | (keys[1:] != keys[:-1])
    run_id = np.cumsum(newrun) - 1
    n_out = int(newrun.sum())
    vals = np.zeros(n_out, dtype=np.float64)
    starts = np.flatnonzero(newrun)
    lens = np.diff(np.append(starts, len(keys)))
    for p in range(int(lens.max()) if n_out else 0):
        live = np.flatnonzero(lens > p)
        vals[live] = vals[live] + prod[starts[live] + p]
    del run_id
    out_rows = rows[starts]
    rowptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(rowptr, out_rows + 1, 1)
    return np.cumsum(rowptr), keys[starts], vals


def csr_ewise(op, ap, aj, av, bp, bj, bv):
    """Element-wise CSR: ``op="add"`` (union; value (0.0 + a) + b, or the one present
    side plus 0.0) or ``op="mul"`` (intersection; value 0.0 + a * b).

    Reference: the two-term union / one-term intersection co-iteration of
    `_run_sparse_output` (engine.py:608-633, `_union_sorted` :224-230,
    `_intersect_sorted` :208-221) with a Workspace slot starting at 0.0 and the
    terms accumulated in expression order (engine.py:594-604).
    """
    ap, aj, bp, bj = (np.asarray(x, dtype=np.int64) for x in (ap, aj, bp, bj))
    av, bv = np.asarray(av, dtype=np.float64), np.asarray(bv, dtype=np.float64)
    m = len(ap) - 1
    n = int(max(aj.max(initial=-1), bj.max(initial=-1))) + 1
    ka = np.repeat(np.arange(m), np.diff(ap)) * n + aj
    kb = np.repeat(np.arange(m), np.diff(bp)) * n + bj
    if op == "mul":
        keys, ia, ib = np.intersect1d(ka, kb, assume_unique=True, return_indices=True)
        vals = 0.0 + av[ia] * bv[ib]
    else:
        keys = np.union1d(ka, kb)
        vals = np.zeros(len(keys), dtype=np.float64)
        pa = np.searchsorted(keys, ka)
        vals[pa] = vals[pa] + av
        pb = np.searchsorted(keys, kb)
        vals[pb] = vals[pb] + bv
    rows = keys // max(n, 1)
    rowptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    return np.cumsum(rowptr), keys % max(n, 1), vals


def relu(x):
    return np.maximum(np.asarray(x, dtype=np.float64), 0.0)


def parity_gate(got, want, bound, rel: float = 1e-5):
    """North-star tolerance: per output row, max |got - want| <= rel * max of the
    row's absolute-value contraction. Returns (ok, worst ratio)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    bound = np.asarray(bound, dtype=np.float64)
    if got.shape != want.shape:
        return False, float("inf")
    if got.size == 0:
        return True, 0.0
    g2 = got.reshape(got.shape[0], -1) if got.ndim > 1 else got.reshape(-1, 1)
    w2 = want.reshape(g2.shape)
    b2 = bound.reshape(g2.shape)
    err = np.abs(g2 - w2).max(axis=1)
    lim = rel * b2.max(axis=1)
    # rows whose bound is 0 must be exact
    ratio = np.where(lim > 0, err / np.where(lim > 0, lim, 1.0), np.where(err > 0, np.inf, 0.0))
    worst = float(ratio.max())
    return worst <= 1.0, worst
