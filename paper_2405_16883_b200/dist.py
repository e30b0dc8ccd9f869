"""Multi-GPU plumbing for the sparse-contraction path.

One process per GPU (torch.distributed, NCCL on GPUs / gloo on CPU). The path
partitions without a data-path exchange: SpMM / SDDMM / softmax / PV shard
rows balanced by nnz with the dense operand replicated (outputs are
row-disjoint), attention shards heads, MTTKRP shards the sorted COO by nnz.
The only real exchange is the GCN's between-layer all-gather of H when one
graph is row-sharded (``allgather_rows``). bench.py's N>1 mode runs
independent per-rank replicas (weak scaling) and reduces the step time with
``max_over_ranks``.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def nnz_balanced_row_shards(rowptr, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges with ~equal (rows + nnz) work each (merge-path split)."""
    rp = np.asarray(rowptr, dtype=np.int64)
    m = len(rp) - 1
    work = rp + np.arange(m + 1)          # merged-sequence position of each row start
    total = work[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(work, r * total / world, side="left")))
    cuts.append(m)
    cuts = np.maximum.accumulate(np.asarray(cuts))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(world)]


def shard_csr(rowptr, colidx, vals, r0: int, r1: int):
    """Local CSR of rows [r0, r1) (column space unchanged: the dense operand is replicated)."""
    rp = np.asarray(rowptr, dtype=np.int64)
    a, b = rp[r0], rp[r1]
    return rp[r0:r1 + 1] - a, np.asarray(colidx)[a:b], np.asarray(vals)[a:b]


def max_over_ranks(x: float, device=None) -> float:
    """Max of a scalar over all ranks (the contract's timing reduction)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allgather_rows(local: torch.Tensor, shards: list[tuple[int, int]]) -> torch.Tensor:
    """Reassemble row shards of a dense result on every rank (the GCN H exchange)."""
    world = dist.get_world_size()
    width = local.shape[1:]
    rows = max(r1 - r0 for r0, r1 in shards)
    padded = torch.zeros((rows,) + tuple(width), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded)
    return torch.cat([b[: r1 - r0] for b, (r0, r1) in zip(bufs, shards)], dim=0)
