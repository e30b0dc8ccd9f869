"""Seeded tensor builders for tests (same recipes as the reference's tests/conftest.py:26-84)."""

from __future__ import annotations

import functools

import numpy as np

import paper_2405_16883_b200 as st
from paper_2405_16883_b200.expr import Add, Mul

MATRIX_FORMATS = ("dense", "csr", "csc", "dcsr", "coo")
VECTOR_LEVELS = ("dense", "compressed", "coordinate")


def vector_format(kind, n):
    lv = {"dense": st.LevelFormat.DENSE, "compressed": st.LevelFormat.COMPRESSED,
          "coordinate": st.LevelFormat.COORDINATE}[kind]
    return st.TensorFormat((n,), (0,), (lv,))


def random_tensor(rng, shape, fmt_name, density, name, integer=False, device=None):
    size = int(np.prod(shape))
    count = max(0, min(size, round(size * density)))
    flat = rng.choice(size, size=count, replace=False)
    coords = np.stack(np.unravel_index(flat, shape), axis=1)
    if integer:
        vals = rng.integers(-3, 4, size=count).astype(np.float64)
    else:
        vals = rng.uniform(-1.0, 1.0, size=count).astype(np.float32).astype(np.float64)
    entries = [(tuple(int(c) for c in co), float(v)) for co, v in zip(coords, vals)]
    fmt = vector_format(fmt_name, shape[0]) if len(shape) == 1 else st.format_by_name(fmt_name, shape)
    return st.build_from_entries(shape, fmt, entries, name=name, device=device)


def random_expression(rng, extent_cap=8, densities=(0.1, 0.5, 1.0), integer=False, device=None, big=None):
    """The reference's random-expression strategy; ``big`` (optional) gives one index an extent
    in [65, big], so tiled loops run several 64-wide blocks."""
    pool = [st.IndexVar(n) for n in ("i", "j", "k")[: rng.integers(1, 4)]]
    ext = {v: int(rng.integers(1, extent_cap + 1)) for v in pool}
    if big:
        ext[pool[int(rng.integers(len(pool)))]] = int(rng.integers(65, big + 1))
    terms = []
    used = set()
    counter = 0
    for _ in range(int(rng.integers(1, 4))):
        accs = []
        for _ in range(int(rng.integers(1, 4))):
            order = int(rng.integers(1, min(2, len(pool)) + 1))
            vs = [pool[i] for i in rng.choice(len(pool), size=order, replace=False)]
            shape = tuple(ext[v] for v in vs)
            fmt_name = str(rng.choice(MATRIX_FORMATS)) if order == 2 else str(rng.choice(VECTOR_LEVELS))
            t = random_tensor(rng, shape, fmt_name, float(rng.choice(densities)), f"T{counter}",
                              integer, device)
            counter += 1
            accs.append(st.Access(t, tuple(vs)))
            used.update(vs)
        terms.append(accs)
    usable = [v for v in pool if v in used]
    n_out = int(rng.integers(1, len(usable) + 1))
    out = [usable[i] for i in rng.choice(len(usable), size=n_out, replace=False)]
    rhs = functools.reduce(Add, (functools.reduce(Mul, t) for t in terms))
    return st.TensorExpr("Out", tuple(out), rhs)


# ---------------------------------------------------------------------------
# Golden fixtures -> our tensors
# ---------------------------------------------------------------------------

def golden_coords(g, prefix):
    """Host expansion of stored levels (mirror of the reference's stored_entries)."""
    shape = tuple(int(s) for s in g[f"{prefix}_shape"])
    modes = tuple(int(m) for m in g[f"{prefix}_modes"])
    kinds = [str(k) for k in g[f"{prefix}_levels"]]
    vals = g[f"{prefix}_vals"]
    order = len(shape)
    if kinds and kinds[0] == "coordinate":
        perm_cols = [g[f"{prefix}_l{k}_crd"].astype(np.int64) for k in range(order)]
    else:
        perm_cols = []
        reps = 1
        for k, kind in enumerate(kinds):
            ext = shape[modes[k]]
            if kind == "dense":
                perm_cols = [np.repeat(c, ext) for c in perm_cols]
                perm_cols.append(np.tile(np.arange(ext), reps))
                reps *= ext
            else:
                pos = g[f"{prefix}_l{k}_pos"]
                perm_cols = [np.repeat(c, np.diff(pos)) for c in perm_cols]
                perm_cols.append(g[f"{prefix}_l{k}_crd"].astype(np.int64))
                reps = len(perm_cols[-1])
    coords = np.zeros((len(vals), order), dtype=np.int64)
    for k, d in enumerate(modes):
        coords[:, d] = perm_cols[k]
    return shape, modes, kinds, coords, vals


def golden_format(shape, modes, kinds):
    lv = {"dense": st.LevelFormat.DENSE, "compressed": st.LevelFormat.COMPRESSED,
          "coordinate": st.LevelFormat.COORDINATE}
    return st.TensorFormat(shape, modes, tuple(lv[k] for k in kinds))


def golden_tensor(g, name, device=None):
    shape, modes, kinds, coords, vals = golden_coords(g, f"in_{name}")
    fmt = golden_format(shape, modes, kinds)
    if all(k == "dense" for k in kinds) and modes == tuple(range(len(shape))):
        return st.from_dense(vals.reshape(shape), name=name, device=device)
    return st.from_arrays(shape, fmt, coords, vals, name=name, device=device, duplicates="error")


def abs_bound(e, tensors):
    """Per-element magnitude bound: the expression over |operands| in float64."""
    import string

    letters = {}
    for v in e.output_indices:
        letters.setdefault(v, string.ascii_letters[len(letters)])
    out = None
    for term in e.terms():
        ops, subs = [], []
        for a in term:
            ops.append(np.abs(st.to_dense(tensors[a.tensor.name])))
            subs.append("".join(letters.setdefault(v, string.ascii_letters[len(letters)]) for v in a.indices))
        term_vars = {v for a in term for v in a.indices}
        present = [v for v in e.output_indices if v in term_vars]
        r = np.einsum(",".join(subs) + "->" + "".join(letters[v] for v in present), *ops)
        if len(present) != len(e.output_indices):  # broadcast over output indices the term lacks
            shape = [s if v in term_vars else 1 for v, s in zip(e.output_indices, e.output_shape)]
            r = np.broadcast_to(r.reshape(shape), e.output_shape)
        out = r if out is None else out + r
    return out
