"""Kernel-level operators on device buffers (thin wrappers over ``libstc.so``).

These are the building blocks the engine's variant dispatch calls; they are
also usable directly (``spmm_csr(rowptr, colidx, vals, B)`` etc.). Every
function launches on ``torch.cuda.current_stream()`` and allocates outputs,
partitions and workspaces with torch (the C ABI never allocates).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import torch

from . import _abi
from ._abi import check, lib, on_operand_device, ptr, require_cuda, stream_handle
from .tensor import ShapeError

# Items (row ends + stored entries) per sub-warp in the merge-path split; 0 means
# "plan it": whole waves of resident CTAs (stc_merge_plan_items_per_group).
DEFAULT_ITEMS_PER_GROUP = int(os.environ.get("STC_ITEMS_PER_GROUP", "0"))
# Row-length skew (max / mean) above which the nnz-balanced split is chosen.
MERGE_SKEW_THRESHOLD = 8.0
# Interleave the entries of rows longer than a merge group (plans built with colidx/vals).
INTERLEAVE = os.environ.get("STC_INTERLEAVE", "1") != "0"
# MTTKRP plans carry prepared items (cp.async-staged kernel); 0 = raw-stream merge kernel (A/B runs)
PREPARED_MTTKRP = os.environ.get("STC_PREPARED_MTTKRP", "1") != "0"
# Dense widths above which the column-tiled variant is chosen.
COLTILE_MIN_K = 512


def _f32(t: torch.Tensor) -> torch.Tensor:
    if t.dtype != torch.float32:
        raise TypeError(f"expected float32, got {t.dtype}")
    return t


def _i32(t: torch.Tensor) -> torch.Tensor:
    if t.dtype != torch.int32:
        raise TypeError(f"expected int32 indices, got {t.dtype}")
    return t


# ---------------------------------------------------------------------------
# Plans (cached per sparse structure, like the reference caches a Schedule)
# ---------------------------------------------------------------------------


@dataclass
class RowStats:
    m: int
    nnz: int
    max_row: int

    @property
    def skew(self) -> float:
        mean = self.nnz / self.m if self.m else 0.0
        return self.max_row / mean if mean > 0 else 0.0


@on_operand_device
def row_stats(rowptr: torch.Tensor) -> RowStats:
    m = rowptr.numel() - 1
    if m <= 0:
        return RowStats(max(m, 0), 0, 0)
    lens = rowptr[1:] - rowptr[:-1]
    mx, nnz = torch.stack([lens.max().long(), rowptr[-1].long()]).tolist()
    return RowStats(m, int(nnz), int(mx))


def choose_variant(stats: RowStats, k: int, aligned: bool = True, n_cols: int | None = None) -> str:
    """The reference's plan for C(i,k)=A(i,j)*B(j,k) is always [i,j,k] with
    tiles {k} (scheduler.py / tiling.py); on the device the same plan splits
    into three variants by the shape of the data.

    COLTILE reads every B row of a column slab once per 224-row block, i.e. B's bytes
    m / 224 times, where the gather variants read nnz rows: it is chosen only for wide
    dense operands when A is dense enough (nnz >= m * n / 128) and its plan fits int32."""
    if k >= COLTILE_MIN_K and aligned and coltile_fits(stats, n_cols):
        return "coltile"
    if stats.skew > MERGE_SKEW_THRESHOLD or stats.max_row > 4096:
        return "merge"
    return "row"


def coltile_fits(stats: RowStats, n_cols: int | None) -> bool:
    """COLTILE pays off (and its plan is addressable) for this matrix: density at least
    1/128 and m * ceil(n / 63) plan slots below 2^31. Without ``n_cols`` (unknown width)
    only the density against the widest possible square operand is not checked."""
    if n_cols is None:
        return True
    m = stats.m
    if m == 0 or n_cols == 0:
        return False
    if m * (-(-n_cols // 63)) >= 2**31 - 1:
        return False
    return stats.nnz * 128 >= m * n_cols


@dataclass
class MergePartition:
    starts: torch.Tensor      # int32 [2 * (n_groups + 1)]
    items_per_group: int
    n_groups: int
    # SpMM plans built with the matrix's colidx / vals: copies in which every row longer
    # than a group has its entries interleaved (see interleave_long_rows), else None.
    colidx: torch.Tensor | None = None
    vals: torch.Tensor | None = None
    m: int = -1               # rows and entries of the structure the plan was built for
    nnz: int = -1
    source: tuple | None = None   # (data_ptr, _version) of the colidx / vals the copies came from
    # MTTKRP plans built with the tensor's (jcrd, kcrd, vals) and the factors' shapes: the
    # entries as prepared 16-byte items (stc_mttkrp_prepare_items) for `items_key` =
    # (n_j, ldb, n_k, ldc); mttkrp_coo3 then runs the cp.async-staged kernel.
    items: torch.Tensor | None = None
    items_key: tuple | None = None
    _ws: dict = field(default_factory=dict, repr=False)

    def check(self, m: int, nnz: int, colidx: torch.Tensor, vals: torch.Tensor) -> None:
        """Raise if this plan was built for another structure (or, for a plan carrying
        interleaved copies of A, for other index / value buffers or since-modified values)."""
        if (self.m, self.nnz) != (m, nnz):
            raise ValueError(f"merge partition built for m={self.m}, nnz={self.nnz}; matrix has m={m}, nnz={nnz}")
        if self.source is not None and self.source != _buffer_id(colidx, vals):
            raise ValueError("merge partition carries interleaved copies of another colidx/vals "
                             "(or of values modified since): rebuild it with merge_partition(..., colidx, vals)")

    def workspace(self, k: int, batch: int, device) -> torch.Tensor | None:
        """Carry workspace for this plan, cached per (k, batch, device, current stream): its
        arrival counters return to zero at the end of every launch, so stream-ordered calls
        reuse it."""
        key = (k, batch, str(device), torch.cuda.current_stream(device).cuda_stream)
        if key not in self._ws:
            self._ws[key] = spmm_workspace(self.m, self.nnz, k, "merge", self.items_per_group, batch, device)
        return self._ws[key]


def _buffer_id(colidx: torch.Tensor, vals: torch.Tensor) -> tuple:
    return (colidx.data_ptr(), colidx._version, vals.data_ptr(), vals._version)


@on_operand_device
def interleave_long_rows(rowptr: torch.Tensor, colidx: torch.Tensor, vals: torch.Tensor, span: int):
    """Copies of (colidx, vals) in which each row longer than ``span`` entries is stored as
    G = ceil(len / span) interleaved sequences (entries 0, G, 2G, ..., then 1, G+1, ...).

    A merge-path group covering part of a long row then gathers columns from the whole
    row's range instead of one contiguous slice of it: sorted columns put a hub row's hot
    (low-index, L2-resident) neighbours first and its cold ones last, so contiguous
    slices finish at very different times (cfg2: 66-100 us for equal work). The row's
    sum is the same up to the summation order (a fixed permutation: deterministic, and
    within the parity gate). Returns (None, None) for an empty matrix."""
    m = rowptr.numel() - 1
    nnz = colidx.numel()
    if m <= 0 or nnz == 0:
        return None, None
    require_cuda(rowptr, colidx, vals)
    ci, va = torch.empty_like(colidx), torch.empty_like(vals)
    check(lib().stc_merge_interleave(m, nnz, ptr(_i32(rowptr)), ptr(_i32(colidx)), ptr(_f32(vals)), int(span),
                                     ptr(ci), ptr(va), stream_handle()), "stc_merge_interleave")
    return ci, va


def plan_items_per_group(m: int, nnz: int, k: int, batch: int = 1, kind: str = "spmm") -> int:
    if kind == "mttkrp_prepared":
        ipg = int(lib().stc_mttkrp_prepared_items_per_group(m, nnz, max(k, 1)))
    else:
        ipg = int(lib().stc_merge_plan_items_per_group(m, nnz, max(k, 1), batch, 1 if kind == "mttkrp" else 0))
    if ipg < 0:
        check(ipg, "stc_merge_plan_items_per_group")
    return ipg


@on_operand_device
def merge_partition(rowptr: torch.Tensor, nnz: int, items_per_group: int | None = None, *,
                    k: int = 128, batch: int = 1, kind: str = "spmm", colidx: torch.Tensor | None = None,
                    vals: torch.Tensor | None = None, max_row: int | None = None,
                    jcrd: torch.Tensor | None = None, kcrd: torch.Tensor | None = None,
                    factors: tuple | None = None) -> MergePartition:
    """Plan-time merge-path partition; ``items_per_group`` None/0 = planned for ``k``.
    With the matrix's ``colidx``/``vals`` (SpMM) the plan also carries their long-row
    interleaved copies, and ``spmm_csr`` reads those; use such a plan only with that matrix.
    ``kind="mttkrp"`` with the tensor's ``jcrd``/``kcrd``/``vals`` and ``factors`` =
    (n_j, ldb, n_k, ldc) also prepares the entries as 16-byte items for the cp.async-staged
    MTTKRP kernel (a 16-byte-per-entry copy of T for those leading dimensions)."""
    require_cuda(rowptr)
    _i32(rowptr)
    m = rowptr.numel() - 1
    prepared = (kind == "mttkrp" and PREPARED_MTTKRP and jcrd is not None and kcrd is not None
                and vals is not None and factors is not None and nnz > 0
                and (factors[0] + 1) * factors[1] < 2**32 and (factors[2] + 1) * factors[3] < 2**32)
    if not items_per_group:
        items_per_group = DEFAULT_ITEMS_PER_GROUP or plan_items_per_group(
            m, nnz, k, batch, "mttkrp_prepared" if prepared else kind)
    groups = int(lib().stc_merge_path_groups(m, nnz, items_per_group))
    starts = torch.empty(2 * (groups + 1), dtype=torch.int32, device=rowptr.device)
    rc = lib().stc_merge_path_partition(m, nnz, ptr(rowptr), items_per_group, ptr(starts),
                                        stream_handle())
    check(rc, "stc_merge_path_partition")
    ci = va = source = None
    if kind == "spmm" and colidx is not None and vals is not None and vals.dim() == 1 and INTERLEAVE and m > 0:
        if max_row is None:
            max_row = int((rowptr[1:] - rowptr[:-1]).max().item())
        if max_row > items_per_group:  # some row spans several groups: interleave (a copy of A)
            ci, va = interleave_long_rows(rowptr, _i32(colidx), _f32(vals), items_per_group)
            source = _buffer_id(colidx, vals)
    items = items_key = None
    if prepared:
        require_cuda(jcrd, kcrd, vals)
        n_j, ldb, n_k, ldc = (int(x) for x in factors)
        items = torch.empty(int(lib().stc_mttkrp_items_bytes(nnz)), dtype=torch.uint8, device=rowptr.device)
        check(lib().stc_mttkrp_prepare_items(nnz, ptr(_i32(jcrd)), ptr(_i32(kcrd)), ptr(_f32(vals)), n_j, ldb,
                                             n_k, ldc, ptr(items), stream_handle()), "stc_mttkrp_prepare_items")
        items_key = (n_j, ldb, n_k, ldc)
        source = (jcrd.data_ptr(), jcrd._version, kcrd.data_ptr(), kcrd._version, vals.data_ptr(), vals._version)
    return MergePartition(starts, items_per_group, groups, ci, va, m, int(nnz), source, items, items_key)


@dataclass
class ColtilePlan:
    """Prepared form of A for the COLTILE variant (int32 buffer, see include/stc.h).

    It carries A's values: build it from the same (rowptr, colidx, vals) the SpMM
    is called with, and rebuild it when the values change. The engine caches it per
    tensor, which is safe because tensors are immutable (`tensor.py:53-56`).
    """

    plan: torch.Tensor
    nnz: int
    m: int = -1               # rows / operand rows of the structure the plan was built for
    n: int = -1
    source: tuple | None = None   # (data_ptr, _version) of the colidx / vals the plan encodes

    def check(self, m: int, n: int, nnz: int, colidx: torch.Tensor, vals: torch.Tensor) -> None:
        """Raise if this plan encodes another matrix: the kernel indexes the plan with the
        call's m and n, and computes with the values stored in the plan."""
        if self.m >= 0 and (self.m, self.n, self.nnz) != (m, n, nnz):
            raise ValueError(f"COLTILE plan built for m={self.m}, n={self.n}, nnz={self.nnz}; "
                             f"matrix has m={m}, n={n}, nnz={nnz}")
        if self.nnz != nnz:
            raise ValueError(f"COLTILE plan built for nnz={self.nnz}, matrix has {nnz}")
        if self.source is not None and self.source != _buffer_id(colidx, vals):
            raise ValueError("COLTILE plan carries the entries of another colidx/vals (or of values "
                             "modified since): rebuild it with coltile_plan(rowptr, colidx, n, vals)")


@on_operand_device
def coltile_plan(rowptr: torch.Tensor, colidx: torch.Tensor, n_cols: int, vals: torch.Tensor) -> ColtilePlan:
    require_cuda(rowptr, colidx, vals)
    m = rowptr.numel() - 1
    nnz = int(colidx.numel())
    ints = int(lib().stc_coltile_plan_ints(m, n_cols, nnz))
    if ints < 0:
        raise ValueError(f"COLTILE plan unsupported for m={m} n={n_cols} nnz={nnz}")
    plan = torch.empty(max(ints, 1), dtype=torch.int32, device=rowptr.device)
    check(lib().stc_coltile_plan(m, n_cols, nnz, ptr(_i32(rowptr)), ptr(_i32(colidx)), ptr(_f32(vals)), ptr(plan),
                                 ints, stream_handle()), "stc_coltile_plan")
    return ColtilePlan(plan, nnz, m, int(n_cols), _buffer_id(colidx, vals))


def spmm_workspace(m: int, nnz: int, k: int, variant: str, items_per_group: int, batch: int,
                   device) -> torch.Tensor | None:
    n = int(lib().stc_spmm_workspace_bytes(m, nnz, k, _abi.VARIANTS[variant], items_per_group, batch))
    if n == 0:
        return None
    # zero once: the arrival counters at its tail must start (and end) at zero
    return torch.zeros((n + 3) // 4, dtype=torch.float32, device=device)


# ---------------------------------------------------------------------------
# SpMM
# ---------------------------------------------------------------------------


@on_operand_device
def spmm_csr(rowptr: torch.Tensor, colidx: torch.Tensor, vals: torch.Tensor, B: torch.Tensor,
             *, out: torch.Tensor | None = None, addend: torch.Tensor | None = None,
             relu: bool = False, variant: str | None = None,
             partition=None, workspace: torch.Tensor | None = None,
             stats: RowStats | None = None) -> torch.Tensor:
    """``C = act(A @ B + addend)`` with A in CSR (int32 rowptr/colidx, fp32 vals).

    ``partition``: a ``MergePartition`` for "merge", a ``ColtilePlan`` for "coltile"
    (computed here when omitted; cache it with the matrix for repeated calls).
    """
    require_cuda(rowptr, colidx, vals, B)
    _i32(rowptr), _i32(colidx), _f32(vals), _f32(B)
    if B.dim() != 2 or B.stride(1) != 1:
        raise ValueError("B must be a 2-D row-major (stride(1) == 1) tensor")
    m = rowptr.numel() - 1
    n, k = B.shape
    nnz = vals.numel()
    if out is None:
        out = torch.empty((m, k), dtype=torch.float32, device=B.device)
    if out.shape != (m, k) or out.stride(1) != 1:
        raise ValueError("out must be an (m, k) row-major tensor")
    if addend is not None and (addend.shape != (m, k) or addend.stride(1) != 1):
        raise ValueError("addend must be an (m, k) row-major tensor")
    if variant is None:
        stats = stats or row_stats(rowptr)
        variant = choose_variant(stats, k, aligned=(k % 4 == 0), n_cols=n)
    v = _abi.VARIANTS[variant]
    ipg = 0
    plan_ptr = None
    if variant == "merge":
        partition = partition or merge_partition(rowptr, nnz, k=k, colidx=colidx, vals=vals,
                                                 max_row=None if stats is None else stats.max_row)
        partition.check(m, nnz, colidx, vals)
        ipg = partition.items_per_group
        plan_ptr = ptr(partition.starts)
        if partition.colidx is not None:   # the plan's long-row interleaved entries
            colidx, vals = partition.colidx, partition.vals
        if workspace is None:
            workspace = partition.workspace(k, 1, B.device)
    elif variant == "coltile":
        partition = partition or coltile_plan(rowptr, colidx, n, vals)
        partition.check(m, n, nnz, colidx, vals)
        plan_ptr = ptr(partition.plan)
    ws_bytes = 0 if workspace is None else workspace.numel() * 4
    rc = lib().stc_spmm_csr_f32(
        m, n, k, ptr(rowptr), ptr(colidx), ptr(vals), nnz, ptr(B), B.stride(0), ptr(out),
        out.stride(0), ptr(addend), 0 if addend is None else addend.stride(0), v,
        _abi.EPILOGUE_RELU if relu else _abi.EPILOGUE_NONE, plan_ptr, ipg, ptr(workspace), ws_bytes,
        stream_handle())
    check(rc, "stc_spmm_csr_f32")
    return out


@on_operand_device
def spmm_csr_batched(rowptr, colidx, vals: torch.Tensor, B: torch.Tensor, *,
                     out: torch.Tensor | None = None, variant: str | None = None,
                     partition: MergePartition | None = None,
                     workspace: torch.Tensor | None = None,
                     stats: RowStats | None = None) -> torch.Tensor:
    """Shared-structure batched SpMM: vals [Z, nnz], B [Z, n, k] -> out [Z, m, k]."""
    require_cuda(rowptr, colidx, vals, B)
    Z, n, k = B.shape
    m = rowptr.numel() - 1
    nnz = colidx.numel()
    if vals.shape != (Z, nnz) or vals.stride(1) != 1 or B.stride(2) != 1:
        raise ValueError("vals must be [Z, nnz] and B [Z, n, k] row-major")
    if out is None:
        out = torch.empty((Z, m, k), dtype=torch.float32, device=B.device)
    if variant is None:
        stats = stats or row_stats(rowptr)
        variant = "merge" if stats.skew > MERGE_SKEW_THRESHOLD else "row"
    if variant == "coltile":
        variant = "row"
    ipg = 0
    if variant == "merge":
        partition = partition or merge_partition(rowptr, nnz, k=k, batch=Z)
        if (partition.m, partition.nnz) != (m, nnz):
            raise ValueError(f"merge partition built for m={partition.m}, nnz={partition.nnz}")
        ipg = partition.items_per_group
        if workspace is None:
            workspace = partition.workspace(k, Z, B.device)
    ws_bytes = 0 if workspace is None else workspace.numel() * 4
    rc = lib().stc_spmm_csr_batched_f32(
        Z, m, n, k, ptr(rowptr), ptr(colidx), ptr(vals), nnz, vals.stride(0), ptr(B), B.stride(1),
        B.stride(0), ptr(out), out.stride(1), out.stride(0), _abi.VARIANTS[variant],
        _abi.EPILOGUE_NONE, None if partition is None else ptr(partition.starts), ipg,
        ptr(workspace), ws_bytes, stream_handle())
    check(rc, "stc_spmm_csr_batched_f32")
    return out


@dataclass
class Segments:
    """Distinct-row segmentation of a sorted COO row column."""

    rows: torch.Tensor     # int32 [n_seg]
    ptr: torch.Tensor      # int32 [n_seg + 1]

    @property
    def n_seg(self) -> int:
        return self.rows.numel()


@on_operand_device
def coo_segments(row_crd: torch.Tensor) -> Segments:
    require_cuda(row_crd)
    _i32(row_crd)
    nnz = row_crd.numel()
    dev = row_crd.device
    seg_rows = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    seg_ptr = torch.empty(nnz + 1, dtype=torch.int32, device=dev)
    n_seg = torch.zeros(1, dtype=torch.int32, device=dev)
    tb = int(lib().stc_coo_segments_temp_bytes(nnz))
    temp = torch.empty(max(tb, 1), dtype=torch.uint8, device=dev)
    rc = lib().stc_coo_segments(nnz, ptr(row_crd), ptr(seg_rows), ptr(seg_ptr), ptr(n_seg), ptr(temp),
                                tb, stream_handle())
    check(rc, "stc_coo_segments")
    s = int(n_seg.item())
    return Segments(seg_rows[:s].clone(), seg_ptr[: s + 1].clone())


def spmm_segments(seg: Segments, colidx: torch.Tensor, vals: torch.Tensor, B: torch.Tensor, *,
                  variant: str | None = None, partition: MergePartition | None = None,
                  workspace: torch.Tensor | None = None) -> torch.Tensor:
    """COO/DCSR SpMM: one output row per segment (the [compressed, dense] output)."""
    return spmm_csr(seg.ptr, colidx, vals, B, variant=variant, partition=partition,
                    workspace=workspace)


# ---------------------------------------------------------------------------
# SDDMM / softmax / attention
# ---------------------------------------------------------------------------


def _head_view(X: torch.Tensor, name: str):
    """(H, rows, d) with unit last stride -> (tensor, head stride, row stride)."""
    if X.dim() == 2:
        X = X.unsqueeze(0)
    if X.dim() != 3 or X.stride(2) != 1:
        raise ValueError(f"{name} must be [rows, d] or [heads, rows, d] with unit last stride")
    return X, X.stride(0) if X.shape[0] > 1 else 0, X.stride(1)


@on_operand_device
def sddmm_csr(rowptr, colidx, Q: torch.Tensor, K: torch.Tensor, *, maskvals=None,
              scale: float = 1.0, out: torch.Tensor | None = None) -> torch.Tensor:
    """``S[h, p] = scale * mask[p] * <Q[h, i], K[h, colidx[p]]>`` -> [H, nnz] (or [nnz])."""
    require_cuda(rowptr, colidx, Q, K)
    squeeze = Q.dim() == 2
    Q3, qhs, qrs = _head_view(_f32(Q), "Q")
    K3, khs, krs = _head_view(_f32(K), "K")
    H, m, d = Q3.shape
    nnz = colidx.numel()
    if out is None:
        out = torch.empty((H, nnz), dtype=torch.float32, device=Q.device)
    rc = lib().stc_sddmm_csr_f32(m, K3.shape[1], d, H, ptr(rowptr), ptr(colidx), ptr(maskvals), nnz,
                                 ptr(Q3), qhs, qrs, ptr(K3), khs, krs, float(scale), ptr(out),
                                 stream_handle())
    check(rc, "stc_sddmm_csr_f32")
    return out[0] if squeeze else out


@on_operand_device
def segment_softmax_(rowptr: torch.Tensor, vals: torch.Tensor) -> torch.Tensor:
    """In-place softmax over each row's stored values; vals [nnz] or [H, nnz]."""
    require_cuda(rowptr, vals)
    v2 = vals.unsqueeze(0) if vals.dim() == 1 else vals
    if not v2.is_contiguous():
        raise ValueError("vals must be contiguous")
    rc = lib().stc_segsoftmax_csr_f32(rowptr.numel() - 1, v2.shape[0], ptr(rowptr), v2.shape[1], ptr(v2),
                                      stream_handle())
    check(rc, "stc_segsoftmax_csr_f32")
    return vals


TILE = 64              # rows per block / columns per tile of the tiled attention path
TILE_MIN_FILL = 1 / 8  # a (block, tile) is dense when it holds at least this share of its slots
TILE_MAX_PER_BLOCK = 8


@dataclass
class AttentionTilePlan:
    """Dense 64x64 mask tiles (+ their values, NaN = absent) and the CSR remainder."""

    tile_cols: torch.Tensor   # int32 [n_blocks, dt_max], -1 padded
    tile_vals: torch.Tensor   # float32 [n_blocks, dt_max, 64, 64]
    rem_rowptr: torch.Tensor  # int32 [m + 1]
    rem_colidx: torch.Tensor  # int32 [rem_nnz]
    rem_vals: torch.Tensor    # float32 [rem_nnz]
    dense_share: float        # fraction of stored entries covered by dense tiles


@on_operand_device
def attention_tile_plan(rowptr: torch.Tensor, colidx: torch.Tensor, maskvals: torch.Tensor | None,
                        n_cols: int, min_fill: float = TILE_MIN_FILL,
                        max_tiles: int = TILE_MAX_PER_BLOCK) -> AttentionTilePlan | None:
    """Plan-time split of a mask into dense 64x64 tiles and a remainder (None if no tile is dense)."""
    require_cuda(rowptr, colidx)
    dev = rowptr.device
    m = rowptr.numel() - 1
    nnz = colidx.numel()
    if m == 0 or nnz == 0:
        return None
    vals = maskvals if maskvals is not None else torch.ones(nnz, dtype=torch.float32, device=dev)
    rows = torch.repeat_interleave(torch.arange(m, device=dev), (rowptr[1:] - rowptr[:-1]).long())
    cols = colidx.long()
    nb, nt = -(-m // TILE), -(-n_cols // TILE)
    blk, tc = rows // TILE, cols // TILE
    counts = torch.bincount(blk * nt + tc, minlength=nb * nt).reshape(nb, nt)
    score = torch.where(counts >= min_fill * TILE * TILE, counts, torch.zeros_like(counts))
    dt = int(min(int((score > 0).sum(1).max().item()), max_tiles))
    if dt == 0:
        return None
    top = torch.topk(score, dt, dim=1)
    valid = top.values > 0
    tsel = torch.where(valid, top.indices, torch.full_like(top.indices, nt))  # invalid sort last
    tsel, order = torch.sort(tsel, dim=1)
    valid = torch.gather(valid, 1, order)
    tile_cols = torch.where(valid, tsel, torch.full_like(tsel, -1)).to(torch.int32)
    slot = torch.full((nb, nt + 1), -1, dtype=torch.long, device=dev)
    bidx = torch.arange(nb, device=dev)[:, None].expand(nb, dt)
    slot[bidx[valid], tsel[valid]] = torch.arange(dt, device=dev)[None, :].expand(nb, dt)[valid]
    s_e = slot[blk, tc]
    inside = s_e >= 0
    tile_vals = torch.full((nb, dt, TILE, TILE), float("nan"), dtype=torch.float32, device=dev)
    tile_vals[blk[inside], s_e[inside], rows[inside] % TILE, cols[inside] % TILE] = vals[inside]
    keep = ~inside
    rem_rowptr = torch.zeros(m + 1, dtype=torch.long, device=dev)
    rem_rowptr[1:] = torch.cumsum(torch.bincount(rows[keep], minlength=m), 0)
    return AttentionTilePlan(tile_cols.contiguous(), tile_vals.contiguous(), rem_rowptr.to(torch.int32),
                             colidx[keep].contiguous(), vals[keep].contiguous(),
                             float(inside.sum().item()) / nnz)


@on_operand_device
def sparse_attention_tiled(plan: AttentionTilePlan, Q, K, V, *, scale: float | None = None,
                           workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Block-tiled fused attention (head dim 64): dense tiles on CUDA cores + remainder."""
    require_cuda(Q, K, V)
    squeeze = Q.dim() == 2
    Q3, qhs, qrs = _head_view(_f32(Q), "Q")
    K3, khs, krs = _head_view(_f32(K), "K")
    V3, vhs, vrs = _head_view(_f32(V), "V")
    H, m, d = Q3.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    nb, dt = plan.tile_cols.shape
    if workspace is None:
        nbytes = int(lib().stc_attention_tiled_workspace_bytes(m, H))
        workspace = torch.empty((nbytes + 3) // 4, dtype=torch.float32, device=Q.device)
    O = torch.empty((H, m, d), dtype=torch.float32, device=Q.device)
    rc = lib().stc_sparse_attention_tiled_f32(
        m, K3.shape[1], d, H, nb, dt, ptr(plan.tile_cols), ptr(plan.tile_vals), ptr(plan.rem_rowptr),
        ptr(plan.rem_colidx), ptr(plan.rem_vals), plan.rem_colidx.numel(), ptr(Q3), qhs, qrs, ptr(K3), khs, krs,
        ptr(V3), vhs, vrs, float(scale), ptr(O), O.stride(0), O.stride(1), ptr(workspace), workspace.numel() * 4,
        stream_handle())
    check(rc, "stc_sparse_attention_tiled_f32")
    return O[0] if squeeze else O


@on_operand_device
def sparse_attention(rowptr, colidx, Q, K, V, *, maskvals=None, scale: float | None = None,
                     return_probs: bool = False):
    """Fused ``O = softmax_rows(scale * M .* QK^T) V``; optionally also S and P [H, nnz]."""
    require_cuda(rowptr, colidx, Q, K, V)
    squeeze = Q.dim() == 2
    Q3, qhs, qrs = _head_view(_f32(Q), "Q")
    K3, khs, krs = _head_view(_f32(K), "K")
    V3, vhs, vrs = _head_view(_f32(V), "V")
    H, m, d = Q3.shape
    nnz = colidx.numel()
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    O = torch.empty((H, m, d), dtype=torch.float32, device=Q.device)
    S = P = None
    if return_probs:
        S = torch.empty((H, nnz), dtype=torch.float32, device=Q.device)
        P = torch.empty((H, nnz), dtype=torch.float32, device=Q.device)
    rc = lib().stc_sparse_attention_f32(
        m, K3.shape[1], d, H, ptr(rowptr), ptr(colidx), ptr(maskvals), nnz, ptr(Q3), qhs, qrs, ptr(K3),
        khs, krs, ptr(V3), vhs, vrs, float(scale), ptr(O), O.stride(0), O.stride(1), ptr(S), ptr(P),
        stream_handle())
    check(rc, "stc_sparse_attention_f32")
    if squeeze:
        O = O[0]
        S = None if S is None else S[0]
        P = None if P is None else P[0]
    return (O, S, P) if return_probs else O


# ---------------------------------------------------------------------------
# MTTKRP
# ---------------------------------------------------------------------------


@on_operand_device
def mttkrp_coo3(seg: Segments, jcrd, kcrd, vals, B: torch.Tensor, C: torch.Tensor, *,
                variant: str = "merge", partition: MergePartition | None = None,
                workspace: torch.Tensor | None = None) -> torch.Tensor:
    """``M[s, :] = sum_{p in segment s} T[p] * B[j[p], :] * C[k[p], :]`` -> [n_seg, R]: per entry
    the term (T[p] * B[j]) * C[k] in entry order (the reference's term order), with B[j, :]
    gathered once per (i, j) fiber."""
    require_cuda(jcrd, kcrd, vals, B, C)
    R = B.shape[1]
    if C.shape[1] != R or B.stride(1) != 1 or C.stride(1) != 1:
        raise ValueError("factor matrices must be row-major with the same rank")
    nnz = vals.numel()
    n_seg = seg.n_seg
    M = torch.empty((n_seg, R), dtype=torch.float32, device=B.device)
    ipg = 0
    key = (B.shape[0], B.stride(0), C.shape[0], C.stride(0))
    if variant == "merge":
        partition = partition or merge_partition(seg.ptr, nnz, k=R, kind="mttkrp", jcrd=jcrd, kcrd=kcrd,
                                                 vals=vals, factors=key)
        if (partition.m, partition.nnz) != (n_seg, nnz):
            raise ValueError(f"merge partition built for m={partition.m}, nnz={partition.nnz}")
        ipg = partition.items_per_group
        if workspace is None:
            workspace = partition.workspace(R, 1, B.device)
    ws_bytes = 0 if workspace is None else workspace.numel() * 4
    if variant == "merge" and partition.items is not None:
        # prepared items: the plan's copy of T for these leading dimensions
        if partition.items_key != key:
            raise ValueError(f"MTTKRP plan prepared for factors (n_j, ldb, n_k, ldc) = {partition.items_key}, "
                             f"called with {key}: rebuild it with merge_partition(..., factors=...)")
        if partition.source != (jcrd.data_ptr(), jcrd._version, kcrd.data_ptr(), kcrd._version,
                                vals.data_ptr(), vals._version):
            raise ValueError("MTTKRP plan carries prepared items of other coordinate / value buffers "
                             "(or of values modified since): rebuild it")
        rc = lib().stc_mttkrp_coo3_prepared_f32(
            n_seg, R, ptr(seg.ptr), ptr(partition.items), nnz, B.shape[0], ptr(B), B.stride(0), C.shape[0],
            ptr(C), C.stride(0), ptr(M), M.stride(0), ptr(partition.starts), ipg, ptr(workspace), ws_bytes,
            stream_handle())
        check(rc, "stc_mttkrp_coo3_prepared_f32")
        return M
    rc = lib().stc_mttkrp_coo3_f32(
        n_seg, R, ptr(seg.ptr), ptr(jcrd), ptr(kcrd), ptr(vals), nnz, B.shape[0], ptr(B), B.stride(0),
        C.shape[0], ptr(C), C.stride(0), ptr(M), M.stride(0), _abi.VARIANTS[variant],
        None if partition is None else ptr(partition.starts), ipg, ptr(workspace), ws_bytes,
        stream_handle())
    check(rc, "stc_mttkrp_coo3_f32")
    return M


# ---------------------------------------------------------------------------
# Sparse x sparse: SpGEMM and element-wise union / product
# ---------------------------------------------------------------------------


@dataclass
class CsrResult:
    """A CSR matrix produced on the device (int32 indices, fp32 values)."""

    rowptr: torch.Tensor
    colidx: torch.Tensor
    vals: torch.Tensor
    products: int = 0   # SpGEMM: number of scalar products (the counter law's P)


def _byte_buffer(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


@on_operand_device
def spgemm_csr(a_rowptr, a_colidx, a_vals, b_rowptr, b_colidx, b_vals, n_cols: int) -> CsrResult:
    """``C(i,k) = A(i,j) * B(j,k)`` for CSR A [m, n], B [n, n_cols] -> CSR C [m, n_cols].

    Every (i,k) reached by a product is stored (arithmetic zeros kept) and each
    value is summed from 0.0 in ascending j, like the reference's workspace
    (engine.py:577-644, 71-90). Two host reads size the outputs.
    """
    a_rowptr, a_colidx, b_rowptr, b_colidx = map(_i32, (a_rowptr, a_colidx, b_rowptr, b_colidx))
    a_vals, b_vals = _f32(a_vals), _f32(b_vals)
    require_cuda(a_rowptr, a_colidx, a_vals, b_rowptr, b_colidx, b_vals)
    m = a_rowptr.numel() - 1
    dev = a_rowptr.device
    L = lib()
    A = (ptr(a_rowptr), ptr(a_colidx), ptr(a_vals))
    B = (ptr(b_rowptr), ptr(b_colidx), ptr(b_vals))
    prod_ptr = torch.empty(m + 1, dtype=torch.int64, device=dev)
    tmp = _byte_buffer(L.stc_spgemm_products_temp_bytes(m), dev)
    check(L.stc_spgemm_products(m, A[0], A[1], B[0], ptr(prod_ptr), ptr(tmp), tmp.numel(), stream_handle()),
          "stc_spgemm_products")
    products = int(prod_ptr[m].item())
    ws_bytes = int(L.stc_spgemm_workspace_bytes(m, n_cols, products))
    if ws_bytes == 0:
        raise ShapeError(f"SpGEMM with {products} products exceeds the int32 range of the device path")
    ws = _byte_buffer(ws_bytes, dev)
    c_rowptr = torch.empty(m + 1, dtype=torch.int32, device=dev)
    check(L.stc_spgemm_symbolic(m, n_cols, *A, *B, ptr(prod_ptr), products, ptr(ws), ws.numel(), ptr(c_rowptr),
                                stream_handle()), "stc_spgemm_symbolic")
    nnz = int(c_rowptr[m].item())
    c_colidx = torch.empty(nnz, dtype=torch.int32, device=dev)
    c_vals = torch.empty(nnz, dtype=torch.float32, device=dev)
    check(L.stc_spgemm_numeric(m, n_cols, *A, *B, products, ptr(ws), ws.numel(), ptr(c_rowptr), ptr(c_colidx),
                               ptr(c_vals), stream_handle()), "stc_spgemm_numeric")
    return CsrResult(c_rowptr, c_colidx, c_vals, products)


@on_operand_device
def csr_ewise(op: str, a_rowptr, a_colidx, a_vals, b_rowptr, b_colidx, b_vals) -> CsrResult:
    """Element-wise CSR of the same shape: ``op="add"`` (union, (0 + a) + b) or
    ``op="mul"`` (intersection, 0 + a * b), the reference's `_union_sorted` /
    `_intersect_sorted` co-iteration (engine.py:208-230)."""
    code = {"add": _abi.EWISE_UNION, "mul": _abi.EWISE_INTERSECT}[op]
    a_rowptr, a_colidx, b_rowptr, b_colidx = map(_i32, (a_rowptr, a_colidx, b_rowptr, b_colidx))
    a_vals, b_vals = _f32(a_vals), _f32(b_vals)
    require_cuda(a_rowptr, a_colidx, a_vals, b_rowptr, b_colidx, b_vals)
    m = a_rowptr.numel() - 1
    if b_rowptr.numel() != m + 1:
        raise ShapeError("element-wise operands need the same number of rows")
    dev = a_rowptr.device
    L = lib()
    c_rowptr = torch.empty(m + 1, dtype=torch.int32, device=dev)
    tmp = _byte_buffer(L.stc_csr_ewise_temp_bytes(m), dev)
    check(L.stc_csr_ewise_symbolic(code, m, ptr(a_rowptr), ptr(a_colidx), ptr(b_rowptr), ptr(b_colidx),
                                   ptr(c_rowptr), ptr(tmp), tmp.numel(), stream_handle()), "stc_csr_ewise_symbolic")
    nnz = int(c_rowptr[m].item())
    c_colidx = torch.empty(nnz, dtype=torch.int32, device=dev)
    c_vals = torch.empty(nnz, dtype=torch.float32, device=dev)
    check(L.stc_csr_ewise_f32(code, m, ptr(a_rowptr), ptr(a_colidx), ptr(a_vals), ptr(b_rowptr), ptr(b_colidx),
                              ptr(b_vals), ptr(c_rowptr), ptr(c_colidx), ptr(c_vals), stream_handle()),
          "stc_csr_ewise_f32")
    return CsrResult(c_rowptr, c_colidx, c_vals)
