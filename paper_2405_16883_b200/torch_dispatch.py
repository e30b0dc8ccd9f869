"""torch.mm / torch.matmul / torch.einsum / ``@`` on declared sparse tensors.

Not in the reference package (its SPEC drops PyTorch interception,
`/root/reference/SPEC.md:16`); the semantics follow the paper's front end
(`/root/reference/PAPER.md:45, 96, 328-330, 430`): a torch call that touches a
declared sparse tensor is desugared into ``parse_einsum`` + ``run``; calls whose
operands are all dense fall through to torch (`PAPER.md:343-345`).

Results of torch-style calls are torch tensors (dense, on the device), like
``torch.sparse.mm``; use ``run``/``execute`` directly to obtain sparse
results in the inferred format.
"""

from __future__ import annotations

import torch

from .expr import parse_einsum
from .tensor import Tensor, from_dense, to_torch

_HANDLED = {}


def _implements(*funcs):
    def deco(fn):
        for f in funcs:
            _HANDLED[f] = fn
        return fn

    return deco


def _wrap(x, name: str) -> Tensor:
    if isinstance(x, Tensor):
        return x
    if torch.is_tensor(x):
        return from_dense(x.detach().to(torch.float32), name=name)
    raise TypeError(f"unsupported operand type {type(x).__name__}")


def _any_sparse(xs) -> bool:
    return any(isinstance(x, Tensor) and x.format.has_sparse_levels for x in xs)


def _plain(x):
    return to_torch(x) if isinstance(x, Tensor) else x


def einsum(equation: str, *operands) -> torch.Tensor:
    if len(operands) == 1 and isinstance(operands[0], (list, tuple)):
        operands = tuple(operands[0])
    if not _any_sparse(operands):
        return torch.einsum(equation, *[_plain(o) for o in operands])
    from .engine import run

    eq = equation.replace(" ", "")
    if "->" not in eq:
        # implicit output: letters appearing exactly once, alphabetical (torch/numpy rule)
        ins = eq.split(",")
        counts = {}
        for g in ins:
            for c in g:
                counts[c] = counts.get(c, 0) + 1
        eq = eq + "->" + "".join(sorted(c for c, n in counts.items() if n == 1))
    tensors = []
    for n, o in enumerate(operands):
        t = _wrap(o, f"T{n}")
        if isinstance(o, torch.Tensor) or t.name in {x.name for x in tensors}:
            t = Tensor(f"T{n}", t.shape, t.storage, t._cache)
        tensors.append(t)
    e = parse_einsum(eq, tensors)
    return to_torch(run(e))


def matmul(a, b) -> torch.Tensor:
    if not _any_sparse((a, b)):
        return torch.matmul(_plain(a), _plain(b))
    ad = a.order if isinstance(a, Tensor) else a.dim()
    bd = b.order if isinstance(b, Tensor) else b.dim()
    if ad == 2 and bd == 2:
        return einsum("ij,jk->ik", a, b)
    if ad == 2 and bd == 1:
        return einsum("ij,j->i", a, b)
    if ad == 1 and bd == 2:
        return einsum("j,jk->k", a, b)
    if ad == 3 and bd == 3:
        return einsum("hij,hjd->hid", a, b)
    raise NotImplementedError(f"matmul of orders {ad} and {bd} with a sparse operand")


def mm(a, b) -> torch.Tensor:
    ad = a.order if isinstance(a, Tensor) else a.dim()
    bd = b.order if isinstance(b, Tensor) else b.dim()
    if ad != 2 or bd != 2:
        raise RuntimeError("mm expects two matrices")
    return matmul(a, b)


_implements(torch.matmul, torch.Tensor.matmul, torch.Tensor.__matmul__)(
    lambda a, b, *args, **kw: matmul(a, b))
_implements(torch.mm, torch.Tensor.mm, torch.sparse.mm)(lambda a, b, *args, **kw: mm(a, b))
_implements(torch.einsum)(lambda eq, *ops, **kw: einsum(eq, *ops))
_implements(torch.Tensor.__rmatmul__)(lambda a, b, *args, **kw: matmul(b, a))


def dispatch_torch_function(func, types, args, kwargs):
    handler = _HANDLED.get(func)
    if handler is None:
        # everything else sees the dense materialisation of our tensors
        args = tuple(_plain(a) for a in args)
        kwargs = {k: _plain(v) for k, v in kwargs.items()}
        return func(*args, **kwargs)
    return handler(*args, **kwargs)
