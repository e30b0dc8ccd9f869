"""Per-configuration measurement on one B200 (all five BASELINE configs).

For each config: GPU time of the hot-path kernel(s) with CUDA events (median
over reps, L2 flushed before every rep), GFLOP/s, compulsory-byte GB/s and the
roofline fraction (HBM for the bandwidth-bound configs, FP32 CUDA-core FMA for
the compute-bound FFN / attention), plus the CPU oracle port timed on this
host (C restatement, all threads) on a bounded sample, extrapolated by nnz.

  python tools/bench_configs.py [--out profiles/configs_r01.json] [--configs 1,2,3,4,5]
"""

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import native, restate  # noqa: E402
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
FLUSH = torch.empty(128 * 1024 * 1024, device="cuda")
PROPS = torch.cuda.get_device_properties(0)


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())["hbm_gbs"], "measured"
    return 6650.0, "fallback"


def fp32_peak_tflops(mhz=1965.0):
    return PROPS.multi_processor_count * 128 * 2 * mhz * 1e6 / 1e12


def gpu_time(fn, reps=20):
    ts = []
    fn()
    torch.cuda.synchronize()
    for _ in range(reps):
        FLUSH.zero_()
        FLUSH.sum()  # read-back: the L2 is left with clean lines (bench.py flush_l2)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def cpu_time(fn, min_s=2.0):
    fn()
    n = 0
    t0 = time.perf_counter()
    while True:
        fn()
        n += 1
        if time.perf_counter() - t0 > min_s:
            break
    return (time.perf_counter() - t0) / n


def dev_csr(A):
    return (torch.from_numpy(A.rowptr).int().cuda(), torch.from_numpy(A.colidx).int().cuda(),
            torch.from_numpy(A.vals).cuda())


def record(name, ms, flops, nbytes, bound, cpu_s, cpu_note, extra=None):
    peak_gbs, kind = hbm_peak()
    gbs = nbytes / (ms * 1e-3) / 1e9
    gf = flops / (ms * 1e-3) / 1e9
    r = {"config": name, "gpu_ms": round(ms, 5), "gflops": round(gf, 1), "compulsory_bytes": int(nbytes),
         "gbs": round(gbs, 1), "frac_hbm_measured": round(gbs / peak_gbs, 4), "frac_hbm_8tbs": round(gbs / 8000, 4),
         "hbm_peak_source": kind, "bound": bound,
         "cpu_oracle_s": round(cpu_s, 4), "cpu_gflops": round(flops / cpu_s / 1e9, 3),
         "cpu_threads": native.num_threads(), "cpu_note": cpu_note, "speedup_vs_cpu_oracle": round(cpu_s * 1e3 / ms, 1)}
    if bound == "fp32":
        r["frac_fp32_peak"] = round(gf / 1e3 / fp32_peak_tflops(), 4)
        r["fp32_peak_tflops"] = round(fp32_peak_tflops(), 1)
    if extra:
        r.update(extra)
    print(json.dumps(r), flush=True)
    return r


def cfg1():
    A, B = synthetic.cfg1()
    R, C, V = dev_csr(A)
    Bt = torch.from_numpy(B).cuda()
    out = torch.empty((A.shape[0], 64), device="cuda")
    stats = ops.row_stats(R)
    variant = ops.choose_variant(stats, 64)
    ms = gpu_time(lambda: ops.spmm_csr(R, C, V, Bt, out=out, variant=variant, stats=stats))
    flops = 2.0 * A.nnz * 64
    nbytes = 4 * (A.shape[0] + 1) + 8 * A.nnz + 2 * 4 * 4096 * 64
    v64, b64 = A.vals.astype(np.float64), B.astype(np.float64)
    cs = cpu_time(lambda: native.spmm_csr(A.rowptr, A.colidx, v64, b64))
    return record("cfg1_csr_spmm_4096_1pct_k64", ms, flops, nbytes, "hbm(L2-resident)", cs, "full",
                  {"variant": variant, "nnz": A.nnz})


def cfg2():
    A, X, W1, W2 = synthetic.cfg2()
    R, C, V = dev_csr(A)
    Z = torch.from_numpy(X).cuda() @ torch.from_numpy(W1).cuda()
    out = torch.empty_like(Z)
    stats = ops.row_stats(R)
    part = ops.merge_partition(R, A.nnz, k=128, colidx=C, vals=V)
    ws = ops.spmm_workspace(A.shape[0], A.nnz, 128, "merge", part.items_per_group, 1, "cuda")
    ms = gpu_time(lambda: ops.spmm_csr(R, C, V, Z, out=out, relu=True, variant="merge", partition=part,
                                       workspace=ws, stats=stats))
    flops = 2.0 * A.nnz * 128
    nbytes = 4 * (A.shape[0] + 1) + 8 * A.nnz + 2 * 4 * A.shape[0] * 128
    z64, v64 = Z.double().cpu().numpy(), A.vals.astype(np.float64)
    cs = cpu_time(lambda: native.spmm_csr(A.rowptr, A.colidx, v64, z64, relu=True))
    return record("cfg2_gcn_spmm_layer_relu", ms, flops, nbytes, "hbm", cs, "full layer",
                  {"variant": "merge", "items_per_group": part.items_per_group, "nnz": A.nnz,
                   "max_row": stats.max_row})


def cfg3():
    W, XT = synthetic.cfg3()
    R, C, V = dev_csr(W)
    Xt = torch.from_numpy(XT).cuda()
    out = torch.empty((W.shape[0], 4096), device="cuda")
    plan = ops.coltile_plan(R, C, 4096, V)  # prepared form of W, cached with the matrix (engine)
    ms = gpu_time(lambda: ops.spmm_csr(R, C, V, Xt, out=out, variant="coltile", partition=plan), reps=10)
    flops = 2.0 * W.nnz * 4096
    nbytes = 4 * (W.shape[0] + 1) + 8 * W.nnz + 4 * 4096 * 4096 + 4 * W.shape[0] * 4096
    v64, x64 = W.vals.astype(np.float64), XT.astype(np.float64)
    rows = 64
    cs = cpu_time(lambda: native.spmm_csr(W.rowptr, W.colidx, v64, x64, rows=(0, rows)), 3.0)
    cs *= W.shape[0] / rows
    return record("cfg3_pruned_ffn_coltile", ms, flops, nbytes, "fp32", cs,
                  f"rows [0,{rows}) extrapolated x{W.shape[0] // rows}", {"variant": "coltile", "nnz": W.nnz})


def cfg4():
    M, Q, K, V = synthetic.cfg4()
    R, C, MV = dev_csr(M)
    Qt, Kt, Vt = (torch.from_numpy(x).cuda() for x in (Q, K, V))
    ms_rows = gpu_time(lambda: ops.sparse_attention(R, C, Qt, Kt, Vt, maskvals=MV, scale=0.125))
    plan = ops.attention_tile_plan(R, C, MV, M.shape[1])
    ws = torch.empty(int(ops.lib().stc_attention_tiled_workspace_bytes(M.shape[0], 16)) // 4, device="cuda")
    ms = gpu_time(lambda: ops.sparse_attention_tiled(plan, Qt, Kt, Vt, scale=0.125, workspace=ws))

    def unfused():
        S = ops.sddmm_csr(R, C, Qt, Kt, maskvals=MV, scale=0.125)
        ops.segment_softmax_(R, S)
        return ops.spmm_csr_batched(R, C, S, Vt)

    ms_unfused = gpu_time(unfused)
    H = 16
    flops = 4.0 * 64 * H * M.nnz
    nbytes = 4 * (M.shape[0] + 1) + 8 * M.nnz + 4 * 4 * H * 8192 * 64
    q64, k64, v64 = Q[0].astype(np.float64), K[0].astype(np.float64), V[0].astype(np.float64)

    def one_head():
        s = 0.125 * native.sddmm_csr(M.rowptr, M.colidx, None, q64, k64)
        p = native.segment_softmax(M.rowptr, s)
        native.spmm_csr(M.rowptr, M.colidx, p, v64)

    cs = cpu_time(one_head) * H
    return record("cfg4_sparse_attention_fused", ms, flops, nbytes, "fp32", cs, "1 head x16",
                  {"kernel": "tiled (dense 64x64 band tiles + remainder)", "per_row_fused_ms": round(ms_rows, 4),
                   "unfused_ms": round(ms_unfused, 4), "nnz_per_head": M.nnz,
                   "dense_tile_share": round(plan.dense_share, 4),
                   "tiles_per_block": int((plan.tile_cols >= 0).sum(1).float().mean().item())})


def cfg5():
    (i, j, k), vals, B, C = synthetic.cfg5()
    It, Jt, Kt = (torch.from_numpy(x).int().cuda() for x in (i, j, k))
    Vt = torch.from_numpy(vals).cuda()
    seg = ops.coo_segments(It)
    Bt, Ct = torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda()
    part = ops.merge_partition(seg.ptr, len(vals), k=32, kind="mttkrp", jcrd=Jt, kcrd=Kt, vals=Vt,
                               factors=(Bt.shape[0], Bt.stride(0), Ct.shape[0], Ct.stride(0)))
    ws = ops.spmm_workspace(seg.n_seg, len(vals), 32, "merge", part.items_per_group, 1, "cuda")
    ms = gpu_time(lambda: ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=part, workspace=ws))
    nnz = len(vals)
    flops = 3.0 * nnz * 32
    nbytes = 16 * nnz + 2 * 4 * 20000 * 32 + 4 * seg.n_seg * 32
    first = np.ones(nnz, bool)
    first[1:] = i[1:] != i[:-1]
    ptr = np.append(np.flatnonzero(first), nnz)
    v64, b64, c64 = vals.astype(np.float64), B.astype(np.float64), C.astype(np.float64)
    cs = cpu_time(lambda: native.mttkrp(ptr, j, k, v64, b64, c64))
    return record("cfg5_mttkrp_zipf_coo3", ms, flops, nbytes, "hbm", cs, "full",
                  {"nnz": nnz, "items_per_group": part.items_per_group, "row0_nnz": int(ptr[1]),
                   "kernel": "prepared items, cp.async-staged" if part.items is not None else "raw streams"})


def spgemm_cfg1():
    """§8(f)-3: SpGEMM A @ A on the cfg1 matrix (CSR x CSR -> CSR, expand-sort-compress)."""
    A, _ = synthetic.cfg1()
    R, C, V = dev_csr(A)
    res = ops.spgemm_csr(R, C, V, R, C, V, A.shape[1])
    P = res.products
    nnz_c = res.vals.numel()
    ms = gpu_time(lambda: ops.spgemm_csr(R, C, V, R, C, V, A.shape[1]))
    flops = 2.0 * P
    nbytes = 2 * (4 * (A.shape[0] + 1) + 8 * A.nnz) + 4 * (A.shape[0] + 1) + 8 * nnz_c
    cs = cpu_time(lambda: restate.spgemm_csr(A.rowptr, A.colidx, A.vals, A.rowptr, A.colidx, A.vals), 3.0)
    return record("x1_spgemm_cfg1_AxA", ms, flops, nbytes, "hbm", cs, "numpy restatement (1 thread)",
                  {"products": P, "nnz_out": nnz_c, "cpu_threads_note": "numpy, single thread"})


def ewise_cfg1():
    """§8(f)-3: element-wise union A + B of two independent cfg1 draws (167k entries each)."""
    A, _ = synthetic.cfg1()
    B, _ = synthetic.cfg1(base=1)  # an independent draw of the same recipe (~1 % overlap)
    R, C, V = dev_csr(A)
    R2, C2, V2 = dev_csr(B)
    res = ops.csr_ewise("add", R, C, V, R2, C2, V2)
    ms = gpu_time(lambda: ops.csr_ewise("add", R, C, V, R2, C2, V2))
    nnz_c = res.vals.numel()
    nbytes = 2 * (4 * (A.shape[0] + 1)) + 8 * (A.nnz + B.nnz) + 4 * (A.shape[0] + 1) + 8 * nnz_c
    cs = cpu_time(lambda: restate.csr_ewise("add", A.rowptr, A.colidx, A.vals, B.rowptr, B.colidx, B.vals), 3.0)
    return record("x2_csr_add_cfg1", ms, float(nnz_c), nbytes, "hbm", cs, "numpy restatement (1 thread)",
                  {"nnz_out": nnz_c})


def walker_ttv_cfg5():
    """Device loop-nest walker (no dedicated kernel) at scale: tensor-times-vector
    y(i,j) = T(i,j,k) * x(k) on the cfg5 tensor (6.55 M entries), through the public API."""
    import paper_2405_16883_b200 as st

    (i, j, k), vals, _, _ = synthetic.cfg5()
    dim = 20000
    T = st.coo_from_sorted_arrays((i, j, k), vals, (dim, dim, dim), name="T")
    xv = np.random.default_rng(3).uniform(0, 1, dim).astype(np.float32)
    x = st.from_dense(torch.from_numpy(xv).cuda(), name="x")
    e = st.parse("y(i,j) = T(i,j,k) * x(k)", {"T": T, "x": x})
    out, _, rep = st.run_with_report(e)
    assert rep["variants"][0].startswith("generic:device-walk"), rep["variants"]
    # parity: float64 fiber sums on the host, structure = the distinct (i, j) fibers
    first = np.ones(len(i), bool)
    first[1:] = (i[1:] != i[:-1]) | (j[1:] != j[:-1])
    starts = np.flatnonzero(first)
    want = np.add.reduceat(vals.astype(np.float64) * xv[k].astype(np.float64), starts)
    got = out.storage.values.cpu().numpy().astype(np.float64)
    assert got.shape == want.shape and np.allclose(got, want, rtol=1e-6, atol=1e-9)
    ms = gpu_time(lambda: st.run(e), reps=5)
    nbytes = 16.0 * len(vals) + 4 * dim + 8 * len(starts)
    v64, x64 = vals.astype(np.float64), xv.astype(np.float64)
    cs = cpu_time(lambda: np.add.reduceat(v64 * x64[k], starts), 2.0)
    return record("x3_walker_ttv_cfg5", ms, 2.0 * len(vals), nbytes, "hbm", cs, "numpy fiber sums (1 thread)",
                  {"nnz": int(len(vals)), "fibers": int(len(starts)), "out_format": out.format.name(),
                   "path": rep["variants"][0][:40]})


def mttkrp_mode2_cfg5():
    """cfg5 tensor, MTTKRP in mode 2 (M(j,r) = T(i,j,k) A(i,r) C(k,r)) through the public API:
    the engine's cached (j, i, k)-sorted view of T feeds the same merge kernel."""
    import paper_2405_16883_b200 as st

    (i, j, k), vals, B, C = synthetic.cfg5()
    dim = 20000
    T = st.coo_from_sorted_arrays((i, j, k), vals, (dim, dim, dim), name="T")
    A = st.from_dense(torch.from_numpy(B).cuda(), name="A")
    Cf = st.from_dense(torch.from_numpy(C).cuda(), name="C")
    e = st.parse("M(j,r) = T(i,j,k) * A(i,r) * C(k,r)", {"T": T, "A": A, "C": Cf})
    out, _, rep = st.run_with_report(e)          # builds and caches the re-sorted view
    api_ms = gpu_time(lambda: st.run(e), reps=10)  # whole public call (host planning included)
    view = T._cache[("mttkrp_view", (1, 0, 2))]
    vst = view.storage
    seg = view._cache[("coo_segments",)]
    part = next(v for kk, v in view._cache.items() if kk[:3] == ("partition", "mttkrp", 32))
    Bd, Cd = torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda()
    ms = gpu_time(lambda: ops.mttkrp_coo3(seg, vst.levels[1].crd, vst.levels[2].crd, vst.values, Bd, Cd,
                                          partition=part))
    nnz = len(vals)
    # parity on a row prefix: the C oracle over the (j, i, k)-sorted entries of j < 200
    order = np.lexsort((k, i, j))
    js, is_, ks, vs = j[order], i[order], k[order], vals[order]
    sel = js < 200
    first = np.ones(sel.sum(), bool)
    first[1:] = js[sel][1:] != js[sel][:-1]
    ptr = np.append(np.flatnonzero(first), sel.sum())
    want = native.mttkrp(ptr, is_[sel], ks[sel], vs[sel], B, C)
    got = out.storage.values.reshape(-1, 32).cpu().numpy()[: len(ptr) - 1]
    assert restate.parity_gate(got, want, want, 1e-5)[0]
    nbytes = 16 * nnz + 2 * 4 * dim * 32 + 4 * dim * 32
    fa = np.ones(nnz, bool)
    fa[1:] = js[1:] != js[:-1]
    ptr_all = np.append(np.flatnonzero(fa), nnz)
    b64, c64, v64 = B.astype(np.float64), C.astype(np.float64), vs.astype(np.float64)
    cs = cpu_time(lambda: native.mttkrp(ptr_all, is_, ks, v64, b64, c64), 2.0)
    return record("x4_mttkrp_mode2_cfg5", ms, 3.0 * nnz * 32, nbytes, "hbm", cs, "full (C oracle, sorted by j)",
                  {"variants": rep["variants"], "nnz": nnz, "public_call_ms": round(api_ms, 3)})


def _wall_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


def construct_cfg5():
    """§8(f)-1: device construction of the cfg5 tensor from its 10 M raw (i, j, k) draws with
    repeats: bounds check, sort, exact duplicate folding (stc_fsum_segments_f64 = math.fsum per
    coordinate), COO assembly. Wall time of from_arrays (host syncs included); CPU: the same
    call on host tensors (torch sort + fsum per repeated group)."""
    import paper_2405_16883_b200 as st

    rng = synthetic.tensor_rng("T")
    i, j, k = (synthetic.truncated_zipf(rng, 10_000_000, 20000, 1.1) for _ in range(3))
    vals = np.random.default_rng(3).uniform(0, 1, len(i))
    coords = np.stack([i, j, k], 1)
    fmt = st.TensorFormat((20000,) * 3, (0, 1, 2), (st.LevelFormat.COORDINATE,) * 3)
    dc, dv = torch.from_numpy(coords).cuda(), torch.from_numpy(vals).cuda()
    ms = _wall_ms(lambda: st.from_arrays((20000,) * 3, fmt, dc, dv, name="T", device="cuda"))
    T = st.from_arrays((20000,) * 3, fmt, dc, dv, name="T", device="cuda")
    t0 = time.perf_counter()
    st.from_arrays((20000,) * 3, fmt, torch.from_numpy(coords), torch.from_numpy(vals), name="T", device="cpu")
    cs = time.perf_counter() - t0
    n = len(vals)
    return record("x5_construct_cfg5_coo_10M", ms, float(n), 24.0 * n + 16.0 * st.nnz(T), "hbm", cs,
                  "same call on host tensors (torch sort + fsum per repeated group, 1 run)",
                  {"entries_in": n, "entries_out": st.nnz(T), "gflops_is": "M entries/ms x 1e-3"})


def construct_cfg2():
    """§8(f)-1: device construction of the cfg2 CSR graph from its symmetrised endpoint list
    (2 m + N entries with repeated edges; values summed exactly)."""
    import paper_2405_16883_b200 as st

    n = 200_000
    rng = synthetic.tensor_rng("A")
    w = (np.arange(n, dtype=np.float64) + 1.0) ** (-1.0 / 1.1)
    w *= 12.0 * n / w.sum()
    m = int(round(w.sum() / 2.0))
    cdf = np.cumsum(w / w.sum())
    cdf[-1] = 1.0
    u = np.searchsorted(cdf, rng.random(m), side="right")
    v = np.searchsorted(cdf, rng.random(m), side="right")
    keep = u != v
    rows = np.concatenate([u[keep], v[keep], np.arange(n)])
    cols = np.concatenate([v[keep], u[keep], np.arange(n)])
    vals = np.random.default_rng(4).uniform(0, 1, rows.size)
    coords = np.stack([rows, cols], 1)
    fmt = st.csr(n, n)
    dc, dv = torch.from_numpy(coords).cuda(), torch.from_numpy(vals).cuda()
    ms = _wall_ms(lambda: st.from_arrays((n, n), fmt, dc, dv, name="A", device="cuda"))
    A = st.from_arrays((n, n), fmt, dc, dv, name="A", device="cuda")
    t0 = time.perf_counter()
    st.from_arrays((n, n), fmt, torch.from_numpy(coords), torch.from_numpy(vals), name="A", device="cpu")
    cs = time.perf_counter() - t0
    return record("x6_construct_cfg2_csr", ms, float(rows.size), 24.0 * rows.size + 8.0 * st.nnz(A), "hbm", cs,
                  "same call on host tensors (torch sort + fsum per repeated group, 1 run)",
                  {"entries_in": int(rows.size), "entries_out": st.nnz(A)})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--configs", default="1,2,3,4,5,x1,x2,x3,x4,x5,x6")
    a = ap.parse_args()
    fns = {"1": cfg1, "2": cfg2, "3": cfg3, "4": cfg4, "5": cfg5, "x1": spgemm_cfg1, "x2": ewise_cfg1,
           "x3": walker_ttv_cfg5, "x4": mttkrp_mode2_cfg5, "x5": construct_cfg5, "x6": construct_cfg2}
    res = [fns[c]() for c in a.configs.split(",")]
    if a.out:
        Path(a.out).write_text(json.dumps({"device": PROPS.name, "sms": PROPS.multi_processor_count,
                                           "results": res}, indent=1))


if __name__ == "__main__":
    main()
