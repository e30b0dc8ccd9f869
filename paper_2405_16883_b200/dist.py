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


class ShardedCSR:
    """This rank's row shard of a CSR matrix, on its own GPU, with a cached SpMM plan.

    The rows are split into ``world`` contiguous ranges of equal rows + nnz work
    (``nnz_balanced_row_shards``); the column space is not split, so the dense operand of an
    SpMM is the full (replicated or all-gathered) matrix and every rank's output rows are its
    own: no reduction across ranks. ``spmm_impl`` replaces the CUDA op (``ops.spmm_csr``)
    only in host-side tests of the partition / exchange logic.
    """

    def __init__(self, rowptr, colidx, vals, shape, rank: int, world: int, device=None, spmm_impl=None):
        self.shape = (int(shape[0]), int(shape[1]))
        self.rank, self.world = rank, world
        self.shards = nnz_balanced_row_shards(rowptr, world)
        self.r0, self.r1 = self.shards[rank]
        rp, ci, v = shard_csr(rowptr, colidx, vals, self.r0, self.r1)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.rowptr = torch.as_tensor(rp).to(dev, torch.int32)
        self.colidx = torch.as_tensor(ci).to(dev, torch.int32)
        self.vals = torch.as_tensor(v).to(dev, torch.float32)
        self._impl = spmm_impl
        self._plan = {}

    @property
    def local_rows(self) -> int:
        return self.r1 - self.r0

    def spmm(self, B: torch.Tensor, relu: bool = False) -> torch.Tensor:
        """Rows [r0, r1) of act(A @ B) for the full dense operand B (n x k)."""
        if B.shape[0] != self.shape[1]:
            raise ValueError(f"dense operand has {B.shape[0]} rows, matrix has {self.shape[1]} columns")
        if self._impl is not None:
            return self._impl(self.rowptr, self.colidx, self.vals, B, relu)
        from . import ops

        k = B.shape[1]
        if k not in self._plan:
            stats = ops.row_stats(self.rowptr)
            variant = ops.choose_variant(stats, k, aligned=k % 4 == 0, n_cols=self.shape[1])
            part = ops.merge_partition(self.rowptr, self.vals.numel(), k=k, colidx=self.colidx, vals=self.vals,
                                       max_row=stats.max_row) if variant == "merge" else None
            self._plan[k] = (stats, variant, part)
        stats, variant, part = self._plan[k]
        return ops.spmm_csr(self.rowptr, self.colidx, self.vals, B, relu=relu, variant=variant, partition=part,
                            stats=stats)


def gcn_forward_sharded(A: ShardedCSR, X_local: torch.Tensor, W1: torch.Tensor, W2: torch.Tensor) -> torch.Tensor:
    """Two-layer GCN forward on a row-sharded graph (configs[1] split over the ranks):
    ``Z1 = X W1`` on local rows -> all-gather Z1 -> ``H = ReLU(A Z1)`` (local rows) ->
    ``Z2 = H W2`` -> all-gather Z2 -> ``O = A Z2`` (local rows). The exchanges move the
    layers' GEMM outputs (n x 128 fp32, NCCL all-gather over NVLink on GPUs) -- the one real
    exchange step of the path; the SpMMs run the CUDA kernels on each rank's shard.
    Returns this rank's rows of O."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        Z1 = _gather(X_local @ W1, A.shards)
        H = A.spmm(Z1, relu=True)
        Z2 = _gather(H @ W2, A.shards)
        return A.spmm(Z2)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def _gather(local: torch.Tensor, shards) -> torch.Tensor:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    return allgather_rows(local, shards)
