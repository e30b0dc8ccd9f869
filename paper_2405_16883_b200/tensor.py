"""Device-resident sparse tensors (drop-in for ``sparsetc.tensor``).

Same logical/physical split as the reference (`/root/reference/pkg/src/sparsetc/tensor.py:24-111`):
a named logical tensor over a ``TensorStorage`` that holds one index structure
per storage level plus a flat array of stored values. What changes is where
and how the buffers live:

* level buffers are ``torch`` tensors on the GPU (``int32`` positions and
  coordinates, ``float32`` values) instead of frozen host ``int64``/``float64``
  numpy arrays (`tensor.py:53-56, 71-72, 205-206`). All configurations of
  this path have fewer than 2**31 stored entries; larger tensors raise.
* construction, conversion and expansion are vectorised torch passes that run
  on whatever device the buffers are on (sort by mode order, run-length the
  compressed levels, cumulative positions), instead of per-segment Python
  loops (`tensor.py:148-219`).
* explicit zeros are stored and duplicates are summed exactly with
  ``math.fsum`` (`tensor.py:222-242`), so the stored structure is bit-identical
  to the reference's for the same entries.

Tensors with storage on the CPU are allowed (planning and format logic are
device independent) but every contraction in ``engine`` requires CUDA storage
and the compiled extension; there is no CPU execution path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .formats import LevelFormat, TensorFormat, dense_format

INDEX_DTYPE = torch.int32
VALUE_DTYPE = torch.float32
_INT32_MAX = 2**31 - 1


class ShapeError(ValueError):
    """Shapes or extents are inconsistent (`tensor.py:20`)."""


def default_device() -> torch.device:
    """CUDA when present; CPU storage is only usable for planning."""
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


def _as_device(device) -> torch.device:
    return default_device() if device is None else torch.device(device)


class StorageArray(torch.Tensor):
    """A storage buffer as the reference exposes it: read-only, numpy-convertible.

    The reference freezes its level arrays (``arr.flags.writeable = False``,
    `tensor.py:53-56, 71-72`), so ``t.storage.values[0] = x`` raises ``ValueError`` and
    ``np.diff(level.pos)`` works. This is a zero-copy alias of the device buffer with the
    same two behaviours: item assignment raises, ``np.asarray`` returns a read-only host
    copy. Torch operations see a plain tensor (``__torch_function__`` is disabled, so
    there is no Python overhead and their results are ordinary tensors); the kernels take
    its ``data_ptr`` as before.
    """

    __torch_function__ = torch._C._disabled_torch_function_impl

    def __setitem__(self, key, value):
        raise ValueError("assignment destination is read-only (tensor storage is immutable)")

    def __array__(self, dtype=None, copy=None):
        a = torch.Tensor.numpy(self.detach().cpu())
        if dtype is not None:
            a = a.astype(dtype, copy=False)
        a.flags.writeable = False
        return a


def _frozen(t: torch.Tensor) -> torch.Tensor:
    return t if type(t) is StorageArray or not isinstance(t, torch.Tensor) else t.as_subclass(StorageArray)


@dataclass(frozen=True)
class DenseLevel:
    extent: int


@dataclass(frozen=True, eq=False)
class CompressedLevel:
    """``pos`` (parents + 1) and ``crd`` (stored coordinates), int32 on device."""

    pos: torch.Tensor
    crd: torch.Tensor

    def __post_init__(self):
        object.__setattr__(self, "pos", _frozen(self.pos))
        object.__setattr__(self, "crd", _frozen(self.crd))


@dataclass(frozen=True, eq=False)
class CoordinateLevel:
    """One column of the aligned coordinate table, int32 on device."""

    crd: torch.Tensor

    def __post_init__(self):
        object.__setattr__(self, "crd", _frozen(self.crd))


LevelData = DenseLevel | CompressedLevel | CoordinateLevel


@dataclass(frozen=True, eq=False)
class TensorStorage:
    format: TensorFormat
    levels: tuple
    values: torch.Tensor

    def __post_init__(self):
        object.__setattr__(self, "values", _frozen(self.values))

    @property
    def device(self) -> torch.device:
        return self.values.device

    def validate(self) -> None:
        """Storage invariants of `tensor.py:67-111`, checked with one host sync."""
        fmt = self.format
        if len(self.levels) != fmt.order:
            raise ValueError("level data arity does not match format")
        if self.values.dtype != VALUE_DTYPE:
            raise ValueError("values must be float32")
        dev = self.values.device
        bad = []  # device booleans, any True -> invalid
        n_positions = 1
        for k, (kind, data) in enumerate(zip(fmt.levels, self.levels)):
            extent = fmt.level_extent(k)
            if kind is LevelFormat.DENSE:
                if not isinstance(data, DenseLevel) or data.extent != extent:
                    raise ValueError(f"level {k}: bad dense level data")
                n_positions *= extent
            elif kind is LevelFormat.COMPRESSED:
                if not isinstance(data, CompressedLevel):
                    raise ValueError(f"level {k}: expected compressed level data")
                pos, crd = data.pos, data.crd
                if pos.dtype != INDEX_DTYPE or crd.dtype != INDEX_DTYPE:
                    raise ValueError(f"level {k}: index buffers must be int32")
                if pos.numel() != n_positions + 1:
                    raise ValueError(f"level {k}: bad positions array")
                pos64 = pos.long()
                bad.append(pos64[0] != 0)
                bad.append(pos64[-1] != crd.numel())
                bad.append((pos64[1:] < pos64[:-1]).any())
                if crd.numel():
                    c = crd.long()
                    bad.append((c < 0).any() | (c >= extent).any())
                    # strictly increasing inside every segment
                    inner = torch.ones(crd.numel(), dtype=torch.bool, device=dev)
                    starts = pos64[:-1][pos64[:-1] < crd.numel()]
                    inner[starts] = False
                    bad.append(((c[1:] <= c[:-1]) & inner[1:]).any())
                n_positions = crd.numel()
            else:
                if not isinstance(data, CoordinateLevel):
                    raise ValueError(f"level {k}: expected coordinate level data")
                if data.crd.numel():
                    c = data.crd.long()
                    bad.append((c < 0).any() | (c >= extent).any())
                n_positions = data.crd.numel()
        if fmt.is_coordinate:
            n = self.levels[0].crd.numel()
            if any(lv.crd.numel() != n for lv in self.levels):
                raise ValueError("coordinate columns differ in length")
            if n > 1:
                cols = [lv.crd.long() for lv in self.levels]
                # tuples strictly increasing in lexicographic order
                gt = torch.zeros(n - 1, dtype=torch.bool, device=dev)
                eq = torch.ones(n - 1, dtype=torch.bool, device=dev)
                for c in cols:
                    gt |= eq & (c[1:] > c[:-1])
                    eq &= c[1:] == c[:-1]
                bad.append(~gt.all())
            n_positions = n
        if self.values.numel() != n_positions:
            raise ValueError(
                f"values length {self.values.numel()} != stored coordinate paths {n_positions}"
            )
        if bad and bool(torch.stack([b.reshape(()) for b in bad]).any().item()):
            raise ValueError("storage violates the format's ordering or range invariants")


@dataclass(frozen=True, eq=False)
class Tensor:
    """Immutable named tensor over device-resident float32 storage (`tensor.py:115-145`).

    Equality is identity, so expressions built over the same tensors compare
    equal exactly like the reference's (whose element-wise array fields are
    only ever compared through the identity shortcut).
    """

    name: str
    shape: tuple
    storage: TensorStorage
    _cache: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        object.__setattr__(self, "shape", tuple(int(s) for s in self.shape))
        if self.storage.format.shape != self.shape:
            raise ShapeError(
                f"storage format shape {self.storage.format.shape} != tensor shape {self.shape}"
            )

    @property
    def format(self) -> TensorFormat:
        return self.storage.format

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.float32)

    @property
    def device(self) -> torch.device:
        return self.storage.device

    @property
    def order(self) -> int:
        return len(self.shape)

    def __repr__(self):
        return (
            f"Tensor({self.name!r}, shape={self.shape}, format={self.format.name()},"
            f" nnz={nnz(self)}, device={self.device})"
        )

    # torch.mm / torch.matmul / torch.einsum / @ interception (see torch_dispatch.py)
    @classmethod
    def __torch_function__(cls, func, types, args=(), kwargs=None):
        from .torch_dispatch import dispatch_torch_function

        return dispatch_torch_function(func, types, args, kwargs or {})

    def __matmul__(self, other):
        from .torch_dispatch import matmul

        return matmul(self, other)

    def __rmatmul__(self, other):
        from .torch_dispatch import matmul

        return matmul(other, self)

    def to(self, device) -> "Tensor":
        """Copy of this tensor with its buffers on ``device``."""
        device = torch.device(device)
        levels = []
        for lv in self.storage.levels:
            if isinstance(lv, CompressedLevel):
                levels.append(CompressedLevel(lv.pos.to(device), lv.crd.to(device)))
            elif isinstance(lv, CoordinateLevel):
                levels.append(CoordinateLevel(lv.crd.to(device)))
            else:
                levels.append(lv)
        st = TensorStorage(self.format, tuple(levels), self.storage.values.to(device))
        return Tensor(self.name, self.shape, st)


# ---------------------------------------------------------------------------
# Assembly: unique entries in logical coordinates -> level buffers
# ---------------------------------------------------------------------------


def _lexsort_rows(cols: list[torch.Tensor], extents: list[int]) -> torch.Tensor:
    """Permutation sorting rows lexicographically by ``cols`` (first = most significant)."""
    n = cols[0].numel() if cols else 0
    dev = cols[0].device if cols else torch.device("cpu")
    if n == 0:
        return torch.zeros(0, dtype=torch.long, device=dev)
    span = 1
    for e in extents:
        span *= e
    if span < 2**62:
        key = torch.zeros(n, dtype=torch.long, device=dev)
        for c, e in zip(cols, extents):
            key = key * e + c
        return torch.sort(key, stable=True).indices
    perm = torch.arange(n, device=dev)
    for c in reversed(cols):
        perm = perm[torch.sort(c[perm], stable=True).indices]
    return perm


def _check_index_range(n: int) -> None:
    if n > _INT32_MAX:
        raise ShapeError(f"{n} stored entries exceed the int32 index range of the device path")


def _assemble_sorted(shape, fmt: TensorFormat, perm_cols: torch.Tensor, vals: torch.Tensor,
                     name: str, validate: bool = True) -> Tensor:
    """Level buffers from unique entries already sorted in storage (mode) order.

    Positional levels are built top-down with vectorised run-length passes:
    a dense level multiplies the parent position by its extent; a compressed
    level keeps one coordinate per distinct (parent, coordinate) pair and its
    positions are the cumulative per-parent counts (`tensor.py:162-219`).
    """
    dev = vals.device
    n = int(vals.numel())
    _check_index_range(n)
    order = fmt.order
    perm_cols = perm_cols.to(torch.long).reshape(n, order)
    vals = vals.to(VALUE_DTYPE)

    if fmt.is_coordinate:
        levels = tuple(CoordinateLevel(perm_cols[:, k].to(INDEX_DTYPE).contiguous()) for k in range(order))
        st = TensorStorage(fmt, levels, vals.contiguous())
        if validate:
            st.validate()
        return Tensor(name, tuple(shape), st)

    parent = torch.zeros(n, dtype=torch.long, device=dev)
    n_pos = 1
    levels = []
    for k, kind in enumerate(fmt.levels):
        extent = fmt.level_extent(k)
        col = perm_cols[:, k]
        if kind is LevelFormat.DENSE:
            parent = parent * extent + col
            n_pos *= extent
            levels.append(DenseLevel(extent))
            continue
        key = parent * extent + col
        first = torch.ones(n, dtype=torch.bool, device=dev)
        if n > 1:
            first[1:] = key[1:] != key[:-1]
        starts = torch.nonzero(first).flatten()
        crd = col[starts]
        counts = torch.bincount(parent[starts], minlength=n_pos) if n else torch.zeros(
            n_pos, dtype=torch.long, device=dev)
        pos = torch.zeros(n_pos + 1, dtype=torch.long, device=dev)
        pos[1:] = torch.cumsum(counts, 0)
        parent = torch.cumsum(first.to(torch.long), 0) - 1
        n_pos = int(starts.numel())
        levels.append(CompressedLevel(pos.to(INDEX_DTYPE), crd.to(INDEX_DTYPE).contiguous()))
    _check_index_range(n_pos)
    if n > 1 and bool((parent[1:] == parent[:-1]).any().item()):
        raise AssertionError("duplicate coordinates survived deduplication")
    out_vals = torch.zeros(n_pos, dtype=VALUE_DTYPE, device=dev)
    if n:
        out_vals[parent] = vals
    st = TensorStorage(fmt, tuple(levels), out_vals)
    if validate:
        st.validate()
    return Tensor(name, tuple(shape), st)


def _assemble(shape, fmt: TensorFormat, coords: torch.Tensor, vals: torch.Tensor, name: str,
              validate: bool = True) -> Tensor:
    """Sort unique logical-order entries by the format's mode order, then assemble."""
    n = int(vals.numel())
    order = fmt.order
    coords = coords.to(torch.long).reshape(n, order)
    perm_cols = coords[:, list(fmt.mode_ordering)] if order else coords
    if n and order:
        extents = [fmt.level_extent(k) for k in range(order)]
        perm = _lexsort_rows([perm_cols[:, k] for k in range(order)], extents)
        perm_cols = perm_cols[perm]
        vals = vals[perm]
    return _assemble_sorted(shape, fmt, perm_cols, vals, name, validate)


# ---------------------------------------------------------------------------
# Public constructors (`tensor.py:222-259`)
# ---------------------------------------------------------------------------


def build_from_entries(shape, fmt: TensorFormat, entries, name: str = "T", device=None) -> Tensor:
    """Tensor from (coordinate tuple, value) pairs.

    Duplicates are summed exactly (``math.fsum``; on a CUDA device by the bit-identical
    ``stc_fsum_segments_f64``), explicit zeros are kept, and the coordinate checks raise
    the reference's exceptions (`tensor.py:222-242`). Values are rounded to float32 once,
    after summation.
    """
    shape = tuple(int(s) for s in shape)
    if fmt.shape != shape:
        raise ShapeError(f"format shape {fmt.shape} != requested shape {shape}")
    coords, vals = [], []
    for coord, value in entries:
        coord = tuple(int(c) for c in coord)
        if len(coord) != len(shape):
            raise ShapeError(f"coordinate {coord} has wrong arity for shape {shape}")
        if any(c < 0 or c >= s for c, s in zip(coord, shape)):
            raise IndexError(f"coordinate {coord} out of bounds for shape {shape}")
        coords.append(coord)
        vals.append(float(value))
    # duplicates summed exactly (fsum per coordinate): on the device when it is CUDA
    return from_arrays(shape, fmt, np.asarray(coords, dtype=np.int64).reshape(len(coords), len(shape)),
                       np.asarray(vals, dtype=np.float64), name, device, duplicates="sum")


def from_arrays(shape, fmt: TensorFormat, coords, values, name: str = "T", device=None,
                duplicates: str = "sum") -> Tensor:
    """Vectorised construction from an (n, order) coordinate array and n values.

    ``duplicates="sum"`` folds repeated coordinates like ``build_from_entries``
    (exact fsum per coordinate, on the device for CUDA storage); ``"error"`` rejects
    them; ``"unique"`` trusts the caller. Runs on ``device`` (default CUDA).
    """
    shape = tuple(int(s) for s in shape)
    if fmt.shape != shape:
        raise ShapeError(f"format shape {fmt.shape} != requested shape {shape}")
    dev = _as_device(device)
    c = torch.as_tensor(np.asarray(coords) if not torch.is_tensor(coords) else coords)
    v = torch.as_tensor(np.asarray(values) if not torch.is_tensor(values) else values)
    n = int(v.numel())
    c = c.to(torch.long).reshape(n, len(shape))
    if n:
        lo = c.min(0).values
        hi = c.max(0).values
        if bool((lo < 0).any()) or any(int(hi[d]) >= shape[d] for d in range(len(shape))):
            raise IndexError(f"coordinates out of bounds for shape {shape}")
    if duplicates != "unique" and n > 1 and not shape:  # order 0: every entry is the same coordinate
        if duplicates == "error":
            raise ValueError("duplicate coordinates")
        c, v = _fold_duplicates(c[:1].expand(n, 0).to(dev), v.to(torch.float64).to(dev),
                                torch.ones(n - 1, dtype=torch.bool, device=dev))
    elif duplicates != "unique" and n > 1:
        perm = _lexsort_rows([c[:, d] for d in range(len(shape))], list(shape))
        cs = c[perm]
        same = (cs[1:] == cs[:-1]).all(1)
        if bool(same.any()):
            if duplicates == "error":
                raise ValueError("duplicate coordinates")
            c, v = _fold_duplicates(cs, v.to(torch.float64)[perm.to(v.device)], same)
    return _assemble(shape, fmt, c.to(dev), v.to(dev).to(VALUE_DTYPE), name)


def _fold_duplicates(cs: torch.Tensor, vs: torch.Tensor, same: torch.Tensor):
    """Sum the values of equal (sorted, adjacent) coordinates exactly, like the reference's
    ``math.fsum`` per coordinate (`tensor.py:238-241`): one float64 result per distinct
    coordinate, correctly rounded. On a CUDA device the groups are summed by
    ``stc_fsum_segments_f64`` (the same algorithm, bit for bit); host tensors use fsum."""
    n = vs.numel()
    first = torch.ones(n, dtype=torch.bool, device=cs.device)
    first[1:] = ~same
    starts = torch.nonzero(first).flatten()
    if cs.is_cuda:
        from . import _abi

        vs = vs.to(cs.device).contiguous()
        bounds = torch.cat([starts, torch.tensor([n], device=cs.device)]).to(torch.int64).contiguous()
        out = torch.empty(starts.numel(), dtype=torch.float64, device=cs.device)
        _abi.check(_abi.lib().stc_fsum_segments_f64(starts.numel(), bounds.data_ptr(), vs.data_ptr(), out.data_ptr(),
                                                    _abi.stream_handle()), "stc_fsum_segments_f64")
        bits = out.view(torch.int64)
        if bool((bits == _abi.FSUM_INF_MINUS_INF).any()):
            raise ValueError("-inf + inf in fsum")
        if bool((bits == _abi.FSUM_OVERFLOW).any()):
            raise OverflowError("intermediate overflow in fsum")
        return cs[starts], out
    v_np = vs.cpu().numpy()
    st_np = starts.cpu().numpy()
    ends = np.append(st_np[1:], n)
    out = v_np[st_np].copy()
    for g in np.flatnonzero(ends - st_np > 1):
        out[g] = math.fsum(v_np[st_np[g]:ends[g]])
    return cs[starts], torch.from_numpy(out)


def csr_from_arrays(rowptr, colidx, values, shape, name: str = "A", device=None,
                    validate: bool = True) -> Tensor:
    """CSR tensor straight from (rowptr, colidx, values) buffers, no re-sorting."""
    dev = _as_device(device)
    nrows, ncols = (int(s) for s in shape)
    pos = torch.as_tensor(rowptr).to(dev, INDEX_DTYPE).contiguous()
    crd = torch.as_tensor(colidx).to(dev, INDEX_DTYPE).contiguous()
    vals = torch.as_tensor(values).to(dev, VALUE_DTYPE).contiguous()
    _check_index_range(int(vals.numel()))
    fmt = TensorFormat((nrows, ncols), (0, 1), (LevelFormat.DENSE, LevelFormat.COMPRESSED))
    st = TensorStorage(fmt, (DenseLevel(nrows), CompressedLevel(pos, crd)), vals)
    if validate:
        st.validate()
    return Tensor(name, (nrows, ncols), st)


def coo_from_sorted_arrays(coords, values, shape, name: str = "T", device=None,
                           validate: bool = True) -> Tensor:
    """All-coordinate tensor from lexicographically sorted, duplicate-free columns."""
    dev = _as_device(device)
    shape = tuple(int(s) for s in shape)
    cols = [torch.as_tensor(c).to(dev, INDEX_DTYPE).contiguous() for c in coords]
    vals = torch.as_tensor(values).to(dev, VALUE_DTYPE).contiguous()
    _check_index_range(int(vals.numel()))
    fmt = TensorFormat(shape, tuple(range(len(shape))), (LevelFormat.COORDINATE,) * len(shape))
    st = TensorStorage(fmt, tuple(CoordinateLevel(c) for c in cols), vals)
    if validate:
        st.validate()
    return Tensor(name, shape, st)


def from_dense(array, fmt: TensorFormat | None = None, name: str = "T", device=None) -> Tensor:
    """Tensor from a dense array (`tensor.py:245-259`).

    All-dense identity formats store every value (zeros included); sparse
    formats keep only the non-zero entries. Torch inputs stay on their
    device unless ``device`` is given; numpy inputs go to the default device.
    """
    if torch.is_tensor(array):
        dev = array.device if device is None else torch.device(device)
        arr = array.detach().to(dev)
    else:
        dev = _as_device(device)
        arr = torch.from_numpy(np.asarray(array, dtype=np.float64)).to(dev)
    shape = tuple(arr.shape)
    if fmt is None:
        fmt = dense_format(shape)
    if fmt.shape != shape:
        raise ShapeError(f"format shape {fmt.shape} != array shape {shape}")
    if fmt.levels and not fmt.has_sparse_levels and fmt.mode_ordering == tuple(range(arr.ndim)):
        st = TensorStorage(
            fmt,
            tuple(DenseLevel(fmt.level_extent(k)) for k in range(fmt.order)),
            arr.reshape(-1).to(VALUE_DTYPE).contiguous().clone(),
        )
        st.validate()
        return Tensor(name, shape, st)
    mask = arr != 0
    coords = torch.nonzero(mask)  # row-major order, unique
    vals = arr[mask]
    return _assemble(shape, fmt, coords, vals.to(VALUE_DTYPE), name)


# ---------------------------------------------------------------------------
# Expansion and conversion (`tensor.py:262-328`)
# ---------------------------------------------------------------------------


def stored_entries_torch(t: Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """All stored coordinate paths (logical order, int64) and values, on device."""
    fmt = t.format
    st = t.storage
    dev = st.device
    n = st.values.numel()
    order = fmt.order
    if fmt.is_coordinate:
        perm_cols = [lv.crd.long() for lv in st.levels]
    else:
        perm_cols: list[torch.Tensor] = []
        reps = 1
        for kind, data in zip(fmt.levels, st.levels):
            if kind is LevelFormat.DENSE:
                e = data.extent
                perm_cols = [c.repeat_interleave(e) for c in perm_cols]
                perm_cols.append(torch.arange(e, device=dev).repeat(reps))
                reps *= e
            else:
                counts = (data.pos[1:].long() - data.pos[:-1].long())
                perm_cols = [c.repeat_interleave(counts) for c in perm_cols]
                perm_cols.append(data.crd.long())
                reps = data.crd.numel()
    coords = torch.zeros((n, order), dtype=torch.long, device=dev)
    for k, dim in enumerate(fmt.mode_ordering):
        coords[:, dim] = perm_cols[k]
    return coords, st.values


def stored_entries(t: Tensor) -> tuple[np.ndarray, np.ndarray]:
    """Host copies: (n, order) int64 coordinates and float64 values (`tensor.py:262`)."""
    coords, vals = stored_entries_torch(t)
    return coords.cpu().numpy(), vals.to(torch.float64).cpu().numpy()


def dense_view(array: torch.Tensor, name: str = "T") -> Tensor:
    """All-dense Tensor over a device torch tensor's own buffer (no copy when it is float32
    and contiguous). For operands of a single call (torch interception), where the
    reference-style copy of ``from_dense`` would cost a full pass over the operand."""
    arr = array.detach()
    if arr.dtype != VALUE_DTYPE or not arr.is_contiguous():
        arr = arr.to(VALUE_DTYPE).contiguous()
    shape = tuple(arr.shape)
    fmt = dense_format(shape)
    st = TensorStorage(fmt, tuple(DenseLevel(fmt.level_extent(k)) for k in range(fmt.order)), arr.reshape(-1))
    return Tensor(name, shape, st)


def to_torch(t: Tensor) -> torch.Tensor:
    """Dense float32 torch tensor on the storage's device; absent entries are 0."""
    fmt = t.format
    if not fmt.has_sparse_levels and fmt.mode_ordering == tuple(range(fmt.order)):
        return t.storage.values.reshape(t.shape).clone()
    out = torch.zeros(t.shape, dtype=VALUE_DTYPE, device=t.device)
    coords, vals = stored_entries_torch(t)
    if vals.numel():
        out[tuple(coords[:, d] for d in range(t.order))] = vals
    return out


def to_dense(t: Tensor) -> np.ndarray:
    """Host float64 array, like the reference's ``to_dense`` (`tensor.py:300`)."""
    return to_torch(t).to(torch.float64).cpu().numpy()


def convert(t: Tensor, target: TensorFormat, name: str | None = None) -> Tensor:
    """Re-store in another format on the tensor's device; no arithmetic (`tensor.py:309`)."""
    if target.shape != t.shape:
        raise ShapeError(f"cannot convert shape {t.shape} to format with shape {target.shape}")
    coords, vals = stored_entries_torch(t)
    return _assemble(t.shape, target, coords, vals, name if name is not None else t.name)


def nnz(t: Tensor) -> int:
    """Number of stored values, explicit zeros included (`tensor.py:321`)."""
    return int(t.storage.values.numel())


def level_is_sparse(fmt: TensorFormat, dim: int) -> bool:
    return fmt.dim_is_sparse(dim)
