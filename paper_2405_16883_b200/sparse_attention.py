"""Sparse attention API: segmented softmax and fused SDDMM -> softmax -> SpMM.

The reference grammar has only ``+`` and ``*`` (`/root/reference/SPEC.md:162-163`),
so its BigBird-style attention (`PAPER.md:282-284, 606-623`) is three separate
expressions and the softmax lives outside the engine. These two entries are the
new API surface for that composition:

* ``segment_softmax(S)`` — row-wise softmax over each row's stored values of a
  CSR (or multi-head ``[dense, dense, compressed]``) tensor; same structure out.
* ``sparse_attention(Q, K, V, mask)`` — O = softmax_rows(scale * M .* QK^T) V in
  one fused kernel (online softmax; S and P never touch HBM unless requested).
"""

from __future__ import annotations

import math

import torch

from . import ops
from .formats import LevelFormat
from .tensor import CompressedLevel, DenseLevel, Tensor, TensorStorage, to_torch


def _rows(t: Tensor):
    f = t.format
    if f.order == 2 and f.mode_ordering == (0, 1) and f.levels == (LevelFormat.DENSE, LevelFormat.COMPRESSED):
        L = t.storage.levels[1]
        return L.pos, L.crd, 1
    if f.order == 3 and f.mode_ordering == (0, 1, 2) and f.levels == (
            LevelFormat.DENSE, LevelFormat.DENSE, LevelFormat.COMPRESSED):
        L = t.storage.levels[2]
        return L.pos, L.crd, t.shape[0]
    raise ValueError(f"segment_softmax needs a CSR or [dense,dense,compressed] tensor, got {f.name()}")


def segment_softmax(S: Tensor, name: str | None = None) -> Tensor:
    """Softmax over every row's stored values; structure (pos/crd) is shared, values are new."""
    pos, _, _ = _rows(S)
    vals = S.storage.values.clone()
    ops.segment_softmax_(pos, vals)
    st = TensorStorage(S.format, S.storage.levels, vals)
    out = Tensor(name or S.name, S.shape, st)
    if "shared_pattern" in S._cache:
        out._cache["shared_pattern"] = S._cache["shared_pattern"]
    return out


def _as_torch(x) -> torch.Tensor:
    return to_torch(x) if isinstance(x, Tensor) else x


def sparse_attention(Q, K, V, mask: Tensor, scale: float | None = None, return_probs: bool = False):
    """Fused sparse attention over a shared CSR mask.

    Q: [M, d] or [H, M, d]; K, V: [N, d] or [H, N, d] (torch CUDA tensors or dense
    Tensors). ``scale`` defaults to 1/sqrt(d). Returns O as a torch tensor; with
    ``return_probs`` also S (scaled scores) and P as [dense, dense, compressed]
    Tensors sharing the mask's pattern.
    """
    f = mask.format
    if not (f.order == 2 and f.mode_ordering == (0, 1) and f.levels == (LevelFormat.DENSE, LevelFormat.COMPRESSED)):
        raise ValueError("sparse_attention needs a CSR mask")
    L = mask.storage.levels[1]
    Qt, Kt, Vt = (_as_torch(x).to(torch.float32).contiguous() for x in (Q, K, V))
    d = Qt.shape[-1]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    if not return_probs and d == ops.TILE:
        # masks with dense bands (local windows) take the block-tiled kernel
        key = ("attention_tile_plan",)
        if key not in mask._cache:
            mask._cache[key] = ops.attention_tile_plan(L.pos, L.crd, mask.storage.values, mask.shape[1])
        plan = mask._cache[key]
        if plan is not None and plan.dense_share >= 0.25:
            return ops.sparse_attention_tiled(plan, Qt, Kt, Vt, scale=scale)
    res = ops.sparse_attention(L.pos, L.crd, Qt, Kt, Vt, maskvals=mask.storage.values, scale=scale,
                               return_probs=return_probs)
    if not return_probs:
        return res
    O, S, P = res
    H = 1 if Qt.dim() == 2 else Qt.shape[0]
    m, n = mask.shape
    nnz = L.crd.numel()
    rp = L.pos.long()
    pos = torch.cat([(rp[:-1][None, :] + torch.arange(H, device=rp.device)[:, None] * nnz).reshape(-1),
                     torch.tensor([H * nnz], device=rp.device)]).to(torch.int32)
    crd = L.crd.repeat(H)
    from .formats import TensorFormat

    fmt = TensorFormat((H, m, n), (0, 1, 2), (LevelFormat.DENSE, LevelFormat.DENSE, LevelFormat.COMPRESSED))
    levels = (DenseLevel(H), DenseLevel(m), CompressedLevel(pos, crd))
    St = Tensor("S", (H, m, n), TensorStorage(fmt, levels, S.reshape(-1)))
    Pt = Tensor("P", (H, m, n), TensorStorage(fmt, levels, P.reshape(-1)))
    for t in (St, Pt):
        t._cache["shared_pattern"] = (L.pos, L.crd)
    return O, St, Pt
