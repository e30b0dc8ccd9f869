"""torch.mm / torch.matmul / torch.einsum / ``@`` on declared sparse tensors.

Not in the reference package (its SPEC drops PyTorch interception,
`/root/reference/SPEC.md:16`); the semantics follow the paper's front end
(`/root/reference/PAPER.md:45, 96, 328-330, 430`): a torch call that touches a
declared sparse tensor is desugared into ``parse_einsum`` + ``run``; calls whose
operands are all dense fall through to torch (`PAPER.md:343-345`).

Results follow the inferred output format (`PAPER.md:328-330`): a dense
inferred output comes back as a torch tensor (like ``torch.sparse.mm``), a
sparse one (SDDMM, multi-head ``[dense, dense, compressed]`` scores, COO/DCSR
SpMM's ``[compressed, dense]`` rows) as the sparse ``Tensor`` itself, never
densified. The parsed expression and its plan are cached per equation and
operand signature (shapes + formats), so a repeated call costs one rebinding.
"""

from __future__ import annotations

from collections import OrderedDict

import torch

from .expr import parse_einsum
from .tensor import Tensor, TensorStorage, dense_view, to_torch

_HANDLED = {}
_EXPRS: OrderedDict = OrderedDict()   # (equation, operand signature) -> parsed expression
_EXPRS_MAX = 64


def _implements(*funcs):
    def deco(fn):
        for f in funcs:
            _HANDLED[f] = fn
        return fn

    return deco


def _any_sparse(xs) -> bool:
    return any(isinstance(x, Tensor) and x.format.has_sparse_levels for x in xs)


def _plain(x):
    return to_torch(x) if isinstance(x, Tensor) else x


def _operand(o, n: int) -> Tensor:
    """Operand n as a Tensor named ``T{n}`` (sparse tensors share storage and plan caches)."""
    if isinstance(o, Tensor):
        return Tensor(f"T{n}", o.shape, o.storage, o._cache)
    if torch.is_tensor(o):
        return dense_view(o, f"T{n}")
    raise TypeError(f"unsupported operand type {type(o).__name__}")


def _placeholder(t: Tensor) -> Tensor:
    return Tensor(t.name, t.shape, TensorStorage(t.format, (), torch.empty(0)))


def _explicit(eq: str) -> str:
    eq = eq.replace(" ", "")
    if "->" in eq:
        return eq
    # implicit output: letters appearing exactly once, alphabetical (torch/numpy rule)
    counts = {}
    for g in eq.split(","):
        for c in g:
            counts[c] = counts.get(c, 0) + 1
    return eq + "->" + "".join(sorted(c for c, n in counts.items() if n == 1))


def einsum(equation: str, *operands):
    """``torch.einsum`` over operands of which at least one is a declared sparse tensor.
    Returns a torch tensor for a dense inferred output, the sparse ``Tensor`` otherwise."""
    if len(operands) == 1 and isinstance(operands[0], (list, tuple)):
        operands = tuple(operands[0])
    if not _any_sparse(operands):
        return torch.einsum(equation, *[_plain(o) for o in operands])
    from .engine import run

    eq = _explicit(equation)
    tensors = [_operand(o, n) for n, o in enumerate(operands)]
    key = (eq, tuple((t.shape, t.format) for t in tensors))
    e = _EXPRS.get(key)
    if e is None:
        # the cached expression holds storage-less placeholders (planning reads only shapes and
        # formats), so the cache keeps no operand buffers alive; every call binds the operands
        e = parse_einsum(eq, [_placeholder(t) for t in tensors])
        _EXPRS[key] = e
        if len(_EXPRS) > _EXPRS_MAX:
            _EXPRS.popitem(last=False)
    else:
        _EXPRS.move_to_end(key)
    result = run(e, {t.name: t for t in tensors})
    if result.format.has_sparse_levels:
        return result
    # a fresh result owns its buffer: hand it out without a copy
    return result.storage.values.reshape(result.shape) if result.format.mode_ordering == tuple(
        range(result.order)) else to_torch(result)


def matmul(a, b):
    """Matrix products return torch tensors, like ``torch.sparse.mm``: an inferred
    ``[compressed, dense]`` output (COO / DCSR / CSC operands) is expanded to its dense rows."""
    if not _any_sparse((a, b)):
        return torch.matmul(_plain(a), _plain(b))
    ad = a.order if isinstance(a, Tensor) else a.dim()
    bd = b.order if isinstance(b, Tensor) else b.dim()
    eq = {(2, 2): "ij,jk->ik", (2, 1): "ij,j->i", (1, 2): "j,jk->k", (3, 3): "hij,hjd->hid"}.get((ad, bd))
    if eq is None:
        raise NotImplementedError(f"matmul of orders {ad} and {bd} with a sparse operand")
    r = einsum(eq, a, b)
    return to_torch(r) if isinstance(r, Tensor) else r


def mm(a, b):
    ad = a.order if isinstance(a, Tensor) else a.dim()
    bd = b.order if isinstance(b, Tensor) else b.dim()
    if ad != 2 or bd != 2:
        raise RuntimeError("mm expects two matrices")
    return matmul(a, b)


def _with_out(fn, name):
    """torch's ``out=`` keyword: the result is copied into ``out`` (dense results only);
    any other keyword is rejected rather than silently dropped."""

    def handler(a, b, *args, out=None, **kw):
        if args or kw:
            raise TypeError(f"{name} on a declared sparse tensor: unsupported arguments "
                            f"{[type(x).__name__ for x in args] + sorted(kw)}")
        r = fn(a, b)
        if out is None:
            return r
        if not torch.is_tensor(r):
            raise TypeError(f"{name}(..., out=) needs a dense result; the inferred output is sparse")
        if out.shape != r.shape:
            raise RuntimeError(f"{name}: out has shape {tuple(out.shape)}, result {tuple(r.shape)}")
        out.copy_(r)
        return out

    return handler


def _einsum_handler(eq, *ops, **kw):
    if kw:
        raise TypeError(f"einsum on a declared sparse tensor: unsupported arguments {sorted(kw)}")
    return einsum(eq, *ops)


_implements(torch.matmul, torch.Tensor.matmul, torch.Tensor.__matmul__)(_with_out(matmul, "matmul"))
_implements(torch.mm, torch.Tensor.mm, torch.sparse.mm)(_with_out(mm, "mm"))
_implements(torch.einsum)(_einsum_handler)
_implements(torch.Tensor.__rmatmul__)(lambda a, b, *args, **kw: _with_out(matmul, "matmul")(b, a, *args, **kw))


def dispatch_torch_function(func, types, args, kwargs):
    handler = _HANDLED.get(func)
    if handler is not None:
        return handler(*args, **(kwargs or {}))
    if _any_sparse(list(args) + list((kwargs or {}).values())):
        # no silent densification of a sparse operand (it may be far larger dense)
        name = getattr(func, "__name__", str(func))
        raise TypeError(f"torch.{name} has no sparse kernel here; densify explicitly with "
                        "to_torch(tensor) or use mm / matmul / einsum / @")
    # all-dense tensors of this package behave as the torch tensors they wrap
    args = tuple(_plain(a) for a in args)
    kwargs = {k: _plain(v) for k, v in (kwargs or {}).items()}
    return func(*args, **kwargs)
