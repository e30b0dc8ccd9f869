"""Dense evaluation of an expression (public ``eval_dense`` of the reference API).

The reference's ``eval_dense`` (`/root/reference/pkg/src/sparsetc/oracle.py:19-46`)
materialises every operand and loops over the full iteration space in Python.
Here the same semantics — every operand densified, each additive term summed
over its own reduction indices, terms added in order — run as one float64
``torch.einsum`` per term on the operands' device. It is an API convenience
for small expressions, not the sparse hot path.
"""

from __future__ import annotations

import string

import numpy as np
import torch

from .expr import TensorExpr
from .tensor import ShapeError, to_torch


def eval_dense(e: TensorExpr, bindings: dict | None = None) -> np.ndarray:
    letters: dict = {}
    for v in e.output_indices:
        letters.setdefault(v, string.ascii_letters[len(letters)])
    out = None
    for term in e.terms():
        operands = []
        subs = []
        for a in term:
            t = a.tensor if bindings is None else bindings.get(a.tensor.name, a.tensor)
            if t.shape != a.tensor.shape:
                raise ShapeError(
                    f"binding for {a.tensor.name} has shape {t.shape}, expected {a.tensor.shape}")
            operands.append(to_torch(t).to(torch.float64))
            subs.append("".join(letters.setdefault(v, string.ascii_letters[len(letters)])
                                for v in a.indices))
        # output indices the term does not mention: the term's value is added at every
        # such coordinate (oracle.py:35-46 loops over all output coordinates)
        term_vars = {v for a in term for v in a.indices}
        present = [v for v in e.output_indices if v in term_vars]
        eq = ",".join(subs) + "->" + "".join(letters[v] for v in present)
        r = torch.einsum(eq, *operands)
        if len(present) != len(e.output_indices):
            shape = [s if v in term_vars else 1 for v, s in zip(e.output_indices, e.output_shape)]
            r = r.reshape(shape).expand(*e.output_shape)
        out = r if out is None else out + r
    return out.cpu().numpy()
