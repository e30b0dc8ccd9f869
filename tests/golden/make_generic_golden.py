"""Golden fixtures for the device loop-nest walker (`paper_2405_16883_b200/generic.py`),
made by running the REAL reference engine on the reference's own random-expression
strategy (`tests/test_acceptance.py:101-116` / conftest recipes, mirrored in
tests/helpers.random_expression). Run in the build container:

    python tests/golden/make_generic_golden.py

For each seed: the expression text, every operand (shape, format, stored entries),
the reference's output storage (format, level pos/crd, values) and its OpCounter
(scalar_mults, scalar_adds, iterator_advances) from ``sparsetc.run_with_report``
(infer_format -> schedule -> tile 64 -> execute).
Output: tests/golden/walk/generic_walk.npz. Nothing here is shipped.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
ROOT = OUT.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2405_16883_b200 as ours  # noqa: E402
from helpers import random_expression  # noqa: E402
from paper_2405_16883_b200.tensor import stored_entries  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
import sparsetc as ref  # noqa: E402
from sparsetc.tensor import CompressedLevel, CoordinateLevel  # noqa: E402

N_CASES = 160
N_TILED = 80


def ref_format(fmt):
    lv = {"dense": ref.LevelFormat.DENSE, "compressed": ref.LevelFormat.COMPRESSED,
          "coordinate": ref.LevelFormat.COORDINATE}
    return ref.TensorFormat(tuple(fmt.shape), tuple(fmt.mode_ordering), tuple(lv[k.value] for k in fmt.levels))


# Hand-written expressions beyond the random strategy's order-2 operands: 3-tensors,
# mixed formats, forced output formats. (source, {name: (shape, format, density)}, out format)
HAND = [
    ("y(i,j) = T(i,j,k) * x(k)", {"T": ((7, 6, 9), "coo", 0.2), "x": ((9,), "dense", 1.0)}, None),
    ("y(i,j) = T(i,j,k) * x(k)", {"T": ((7, 6, 9), "coo", 0.2), "x": ((9,), "compressed", 0.5)}, None),
    ("Y(i,j,r) = T(i,j,k) * C(k,r)", {"T": ((6, 5, 8), "coo", 0.25), "C": ((8, 4), "dense", 1.0)}, None),
    ("M(i,r) = T(i,j,k) * B(j,r) * C(k,r)", {"T": ((9, 7, 8), "coo", 0.15), "B": ((7, 3), "dense", 1.0),
                                              "C": ((8, 3), "dense", 1.0)}, "csr"),
    ("y(i) = A(i,j) * B(i,j)", {"A": ((8, 9), "csr", 0.3), "B": ((8, 9), "coo", 0.4)}, None),
    ("C(i,j) = A(i,j) * B(i,j) + D(i,j)", {"A": ((7, 8), "csr", 0.4), "B": ((7, 8), "csc", 0.4),
                                           "D": ((7, 8), "dcsr", 0.2)}, None),
    ("C(i,j) = A(i,j) + B(j,i)", {"A": ((6, 6), "csr", 0.3), "B": ((6, 6), "csr", 0.3)}, None),
    ("C(i,k) = A(i,j) * B(j,k)", {"A": ((9, 7), "dcsr", 0.3), "B": ((7, 8), "dcsr", 0.3)}, None),
    ("C(i,k) = A(i,j) * B(j,k)", {"A": ((9, 7), "coo", 0.3), "B": ((7, 8), "csc", 0.3)}, None),
    ("C(i,k) = A(i,j) * B(j,k)", {"A": ((9, 7), "csr", 0.3), "B": ((7, 8), "dense", 1.0)}, "dcsr"),
    ("C(k,i) = A(i,j) * B(j,k)", {"A": ((9, 7), "csr", 0.3), "B": ((7, 8), "dense", 1.0)}, "csr"),
    ("y(j) = A(i,j) * x(i)", {"A": ((30, 25), "csr", 0.1), "x": ((30,), "compressed", 0.3)}, None),
    ("y(i) = A(i,j) * x(j) + z(i)", {"A": ((30, 25), "dcsr", 0.1), "x": ((25,), "dense", 1.0),
                                     "z": ((30,), "coordinate", 0.2)}, None),
    ("O(h,i,d) = P(h,i,j) * V(h,j,d)", {"P": ((2, 6, 7), "coo", 0.3), "V": ((2, 7, 4), "dense", 1.0)}, None),
    ("S(h,i,j) = M(i,j) * Q(h,i,d) * K(h,j,d)", {"M": ((6, 7), "dcsr", 0.3), "Q": ((2, 6, 5), "dense", 1.0),
                                                 "K": ((2, 7, 5), "dense", 1.0)}, None),
    ("A2(i,j) = A(i,j) * A(i,j)", {"A": ((8, 8), "coo", 0.3)}, None),
    ("x2(i) = x(i) * y(i) * z(i)", {"x": ((40,), "compressed", 0.5), "y": ((40,), "coordinate", 0.5),
                                     "z": ((40,), "compressed", 0.5)}, None),
    ("x2(i) = x(i) + y(i) + z(i)", {"x": ((40,), "compressed", 0.2), "y": ((40,), "coordinate", 0.2),
                                     "z": ((40,), "dense", 1.0)}, None),
    ("G(i,j) = x(i) * y(j)", {"x": ((9,), "compressed", 0.4), "y": ((8,), "coordinate", 0.4)}, None),
]


def ref_tensor_fmt(fmt_name, shape):
    if len(shape) == 1:
        return ref.TensorFormat(shape, (0,), ({"dense": ref.LevelFormat.DENSE,
                                                "compressed": ref.LevelFormat.COMPRESSED,
                                                "coordinate": ref.LevelFormat.COORDINATE}[fmt_name],))
    if fmt_name == "coo":
        return ref.coo(*shape)
    if fmt_name == "dense":
        return ref.dense_format(shape)
    return ref.format_by_name(fmt_name, shape)


def hand_case(idx, src, spec, out_name, arrays, texts):
    rng = np.random.default_rng(9000 + idx)
    bindings, names = {}, []
    for name, (shape, fmt_name, dens) in spec.items():
        size = int(np.prod(shape))
        count = max(1, round(size * dens))
        flat = np.sort(rng.choice(size, size=count, replace=False))
        coords = np.stack(np.unravel_index(flat, shape), axis=1).astype(np.int64).reshape(count, len(shape))
        vals = rng.uniform(-1, 1, count).astype(np.float32).astype(np.float64)
        fmt = ref_tensor_fmt(fmt_name, shape)
        entries = [(tuple(int(c) for c in co), float(v)) for co, v in zip(coords, vals)]
        bindings[name] = ref.build_from_entries(shape, fmt, entries, name=name)
        p = f"c{idx}_{name}"
        arrays[p + "_coords"] = coords
        arrays[p + "_vals"] = vals
        arrays[p + "_shape"] = np.asarray(shape, dtype=np.int64)
        arrays[p + "_modes"] = np.asarray(fmt.mode_ordering, dtype=np.int64)
        arrays[p + "_levels"] = np.asarray([k.value for k in fmt.levels])
        names.append(name)
    e = ref.parse(src, bindings)
    out_fmt = None if out_name is None else ref.format_by_name(out_name, e.output_shape)
    out, cnt, rep = ref.run_with_report(e, out_format=out_fmt)
    store_out(idx, out, arrays)
    store_counters(idx, cnt, arrays)
    texts.append(src + " | " + ",".join(names) + " | " + rep["path"] + (f" | {out_name}" if out_name else ""))


def store_counters(idx, cnt, arrays):
    """The reference interpreter's OpCounter (engine.py:51-68); None on the dense path."""
    if cnt is not None:
        arrays[f"c{idx}_counters"] = np.asarray([cnt.scalar_mults, cnt.scalar_adds, cnt.iterator_advances],
                                                dtype=np.int64)


def store_out(idx, out, arrays):
    q = f"c{idx}_out"
    for k, lv in enumerate(out.storage.levels):
        if isinstance(lv, CompressedLevel):
            arrays[f"{q}_l{k}_pos"] = np.asarray(lv.pos)
            arrays[f"{q}_l{k}_crd"] = np.asarray(lv.crd)
        elif isinstance(lv, CoordinateLevel):
            arrays[f"{q}_l{k}_crd"] = np.asarray(lv.crd)
    arrays[q + "_vals"] = np.asarray(out.storage.values)
    arrays[q + "_shape"] = np.asarray(out.shape, dtype=np.int64)
    arrays[q + "_modes"] = np.asarray(out.format.mode_ordering, dtype=np.int64)
    arrays[q + "_levels"] = np.asarray([lv.value for lv in out.format.levels])


def main():
    arrays = {}
    texts = []
    random_cases(arrays, texts, N_CASES, 5000, {})
    for h, (src, spec, out_name) in enumerate(HAND):
        hand_case(N_CASES + h, src, spec, out_name, arrays, texts)
    arrays["cases"] = np.asarray(texts)
    np.savez_compressed(OUT / "walk" / "generic_walk.npz", **arrays)
    print(f"{N_CASES} cases -> {OUT / 'walk' / 'generic_walk.npz'}")
    # tiled loops with several 64-wide blocks (one index extent in [65, 140]; only seeds whose
    # plan tiles that index are kept)
    arrays, texts = {}, []
    random_cases(arrays, texts, N_TILED, 7000, {"big": 140, "densities": (0.05, 0.2, 1.0)}, multi_block=True)
    arrays["cases"] = np.asarray(texts)
    np.savez_compressed(OUT / "walk" / "generic_walk_tiled.npz", **arrays)
    print(f"{N_TILED} cases -> {OUT / 'walk' / 'generic_walk_tiled.npz'}")


def _multi_block(e) -> bool:
    from paper_2405_16883_b200.expr import index_extents

    s = ours.tile(e, ours.schedule(e, ours.infer_format(e)), 64)
    ext = index_extents(e)
    return any(ext[v] > 64 for v in s.tiles)


def random_cases(arrays, texts, n_cases, seed0, kw, multi_block=False):
    seed, idx = seed0 - 1, -1
    while idx + 1 < n_cases:
        seed += 1
        rng = np.random.default_rng(seed)
        e = random_expression(rng, extent_cap=6, device="cpu", **kw)
        if multi_block and not _multi_block(e):
            continue
        src = ours.render(e)
        bindings = {}
        names = []
        per_tensor = []
        for a in e.accesses:
            t = a.tensor
            if t.name in bindings:
                continue
            coords, vals = stored_entries(t)
            entries = [(tuple(int(c) for c in co), float(v)) for co, v in zip(coords, vals)]
            bindings[t.name] = ref.build_from_entries(t.shape, ref_format(t.format), entries, name=t.name)
            per_tensor.append((t, coords, vals))
            names.append(t.name)
        re = ref.parse(src, bindings)
        try:
            out, cnt, rep = ref.run_with_report(re)
        except IndexError:
            # the reference's vectorised dense tail indexes past its loop list when the head
            # ends in a tile block (engine.py:405, 555-565); such expressions are not fixtures
            continue
        idx += 1
        for t, coords, vals in per_tensor:
            p = f"c{idx}_{t.name}"
            arrays[p + "_coords"] = np.asarray(coords, dtype=np.int64).reshape(len(vals), len(t.shape))
            arrays[p + "_vals"] = np.asarray(vals, dtype=np.float64)
            arrays[p + "_shape"] = np.asarray(t.shape, dtype=np.int64)
            arrays[p + "_modes"] = np.asarray(t.format.mode_ordering, dtype=np.int64)
            arrays[p + "_levels"] = np.asarray([k.value for k in t.format.levels])
        store_counters(idx, cnt, arrays)
        q = f"c{idx}_out"
        for k, lv in enumerate(out.storage.levels):
            if isinstance(lv, CompressedLevel):
                arrays[f"{q}_l{k}_pos"] = np.asarray(lv.pos)
                arrays[f"{q}_l{k}_crd"] = np.asarray(lv.crd)
            elif isinstance(lv, CoordinateLevel):
                arrays[f"{q}_l{k}_crd"] = np.asarray(lv.crd)
        arrays[q + "_vals"] = np.asarray(out.storage.values)
        arrays[q + "_shape"] = np.asarray(out.shape, dtype=np.int64)
        arrays[q + "_modes"] = np.asarray(out.format.mode_ordering, dtype=np.int64)
        arrays[q + "_levels"] = np.asarray([lv.value for lv in out.format.levels])
        texts.append(src + " | " + ",".join(names) + " | " + rep["path"])


if __name__ == "__main__":
    main()
