"""Seeded synthetic inputs for the five BASELINE configurations.

Seeding follows the reference CLI's convention: each named tensor gets its own
``numpy.random.default_rng((base + crc32(name)) % 2**32)``
(`/root/reference/pkg/src/sparsetc/cli.py:34-35`). Values are drawn in float64
and rounded to float32 once; the same rounded values feed the GPU and the
float64 CPU oracle. Every generator takes size parameters so tests can build
small instances with the same recipe; defaults are the configuration sizes.
All outputs are host numpy arrays (int64 structure, float32 values).
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass

import numpy as np


def tensor_rng(name: str, base: int = 0) -> np.random.Generator:
    return np.random.default_rng((base + zlib.crc32(name.encode())) % (2**32))


def f32(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64).astype(np.float32)


@dataclass
class CSRArrays:
    shape: tuple
    rowptr: np.ndarray   # int64 [m+1]
    colidx: np.ndarray   # int64 [nnz]
    vals: np.ndarray     # float32 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.colidx.size)


def _rowptr_from_counts(counts) -> np.ndarray:
    rp = np.zeros(len(counts) + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    return rp


# ---------------------------------------------------------------------------
# cfg1: uniform-random CSR SpMM
# ---------------------------------------------------------------------------


def uniform_csr(n_rows=4096, n_cols=4096, density=0.01, name="A", base=0) -> CSRArrays:
    """Row nnz ~ Binomial(n_cols, density); columns drawn without replacement per row."""
    rng = tensor_rng(name, base)
    counts = rng.binomial(n_cols, density, size=n_rows)
    cols = [np.sort(rng.choice(n_cols, size=int(c), replace=False)) for c in counts]
    colidx = np.concatenate(cols).astype(np.int64) if n_rows else np.zeros(0, np.int64)
    vals = f32(rng.uniform(-1.0, 1.0, size=colidx.size))
    return CSRArrays((n_rows, n_cols), _rowptr_from_counts(counts), colidx, vals)


def dense_uniform(shape, name, lo=-1.0, hi=1.0, base=0) -> np.ndarray:
    return f32(tensor_rng(name, base).uniform(lo, hi, size=shape))


def dense_normal(shape, name, std=1.0, base=0) -> np.ndarray:
    return f32(tensor_rng(name, base).standard_normal(size=shape) * std)


def cfg1(base=0, n=4096, k=64, density=0.01):
    A = uniform_csr(n, n, density, "A", base)
    B = dense_uniform((n, k), "B", base=base)
    return A, B


# ---------------------------------------------------------------------------
# cfg2: Chung-Lu power-law graph, normalised adjacency, 2-layer GCN
# ---------------------------------------------------------------------------


def chung_lu_adjacency(n=200_000, mean_degree=12.0, exponent=2.1, name="A", base=0) -> CSRArrays:
    """Symmetrised Chung-Lu graph with self loops, values D^-1/2 (A+I) D^-1/2.

    w_i = (i+1)^(-1/(exponent-1)) scaled to mean ``mean_degree``; m = round(sum w / 2)
    endpoint pairs drawn independently with probability proportional to w;
    self pairs dropped, both directions stored, duplicates removed, then I added.
    (Dedupe makes the realised mean degree slightly lower than requested; the
    shortfall is kept, as pinned in SURVEY.md §8(d).)
    """
    rng = tensor_rng(name, base)
    w = (np.arange(n, dtype=np.float64) + 1.0) ** (-1.0 / (exponent - 1.0))
    w *= mean_degree * n / w.sum()
    m = int(round(w.sum() / 2.0))
    p = w / w.sum()
    cdf = np.cumsum(p)
    cdf[-1] = 1.0
    u = np.searchsorted(cdf, rng.random(m), side="right")
    v = np.searchsorted(cdf, rng.random(m), side="right")
    keep = u != v
    u, v = u[keep], v[keep]
    rows = np.concatenate([u, v, np.arange(n)])
    cols = np.concatenate([v, u, np.arange(n)])
    key = np.unique(rows.astype(np.int64) * n + cols)
    rows = key // n
    cols = key % n
    counts = np.bincount(rows, minlength=n)
    dinv = 1.0 / np.sqrt(counts.astype(np.float64))
    vals = f32(dinv[rows] * dinv[cols])
    return CSRArrays((n, n), _rowptr_from_counts(counts), cols.astype(np.int64), vals)


def glorot(fan_in, fan_out, name, base=0) -> np.ndarray:
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    return f32(tensor_rng(name, base).uniform(-lim, lim, size=(fan_in, fan_out)))


def cfg2(base=0, n=200_000, feat=128, mean_degree=12.0):
    A = chung_lu_adjacency(n, mean_degree, 2.1, "A", base)
    X = dense_normal((n, feat), "X", base=base)
    W1 = glorot(feat, feat, "W1", base)
    W2 = glorot(feat, feat, "W2", base)
    return A, X, W1, W2


# ---------------------------------------------------------------------------
# cfg3: magnitude-pruned FFN weight (Y^T = W X^T)
# ---------------------------------------------------------------------------


def pruned_weight(rows=16384, cols=4096, keep_frac=0.1, name="W", base=0) -> CSRArrays:
    rng = tensor_rng(name, base)
    k = int(round(keep_frac * cols))
    rowptr = np.arange(rows + 1, dtype=np.int64) * k
    colidx = np.empty(rows * k, dtype=np.int64)
    vals = np.empty(rows * k, dtype=np.float32)
    chunk = 1024
    for r0 in range(0, rows, chunk):
        W = rng.standard_normal(size=(min(chunk, rows - r0), cols)) * 0.02
        idx = np.argpartition(-np.abs(W), k - 1, axis=1)[:, :k]
        idx.sort(axis=1)
        sl = slice(r0 * k, (r0 + W.shape[0]) * k)
        colidx[sl] = idx.reshape(-1)
        vals[sl] = f32(np.take_along_axis(W, idx, axis=1)).reshape(-1)
    return CSRArrays((rows, cols), rowptr, colidx, vals)


def cfg3(base=0, rows=16384, cols=4096, tokens=4096):
    W = pruned_weight(rows, cols, 0.1, "W", base)
    X = dense_normal((tokens, cols), "X", base=base)
    XT = np.ascontiguousarray(X.T)
    return W, XT


# ---------------------------------------------------------------------------
# cfg4: causal local window + random earlier positions, 16 heads
# ---------------------------------------------------------------------------


def attention_mask(seq=8192, window=256, n_random=64, name="M", base=0) -> CSRArrays:
    rng = tensor_rng(name, base)
    cols_per_row = []
    for q in range(seq):
        win = np.arange(max(0, q - window + 1), q + 1)
        if q > 0:
            rnd = rng.integers(0, q, size=n_random)
            c = np.union1d(win, rnd)
        else:
            c = win
        cols_per_row.append(c)
    counts = np.array([len(c) for c in cols_per_row])
    colidx = np.concatenate(cols_per_row).astype(np.int64)
    vals = np.ones(colidx.size, dtype=np.float32)
    return CSRArrays((seq, seq), _rowptr_from_counts(counts), colidx, vals)


def cfg4(base=0, seq=8192, heads=16, dim=64, window=256, n_random=64):
    M = attention_mask(seq, window, n_random, "M", base)
    Q = dense_normal((heads, seq, dim), "Q", base=base)
    K = dense_normal((heads, seq, dim), "K", base=base)
    V = dense_normal((heads, seq, dim), "V", base=base)
    return M, Q, K, V


# ---------------------------------------------------------------------------
# cfg5: Zipf COO 3-tensor MTTKRP
# ---------------------------------------------------------------------------


def truncated_zipf(rng, n_draws, support=20000, s=1.1) -> np.ndarray:
    """Inverse-CDF draws from P(x) ~ x^-s on {1..support}, returned minus 1."""
    pmf = np.arange(1, support + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(pmf)
    cdf /= cdf[-1]
    return np.searchsorted(cdf, rng.random(n_draws), side="right").astype(np.int64)


def zipf_coo3(dim=20000, n_draws=10_000_000, s=1.1, name="T", base=0):
    """Sorted, duplicate-free COO coordinates (duplicates dropped, not summed)."""
    rng = tensor_rng(name, base)
    i = truncated_zipf(rng, n_draws, dim, s)
    j = truncated_zipf(rng, n_draws, dim, s)
    k = truncated_zipf(rng, n_draws, dim, s)
    key = np.unique((i * dim + j) * dim + k)
    vals = f32(rng.uniform(0.0, 1.0, size=key.size))
    ii = key // (dim * dim)
    jj = (key // dim) % dim
    kk = key % dim
    return (ii, jj, kk), vals


def cfg5(base=0, dim=20000, n_draws=10_000_000, rank=32):
    coords, vals = zipf_coo3(dim, n_draws, 1.1, "T", base)
    B = dense_uniform((dim, rank), "B", 0.0, 1.0, base)
    C = dense_uniform((dim, rank), "C", 0.0, 1.0, base)
    return coords, vals, B, C
