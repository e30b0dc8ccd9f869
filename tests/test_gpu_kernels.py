"""Kernel-level parity on the B200: every variant, shape edge cases, determinism.

Checked against the C oracle (float64, reference summation order) with the
north-star gate: per output row, max |gpu - oracle| <= 1e-5 * max of the
row's absolute-value contraction (|A| @ |B| etc.).
"""

import numpy as np
import pytest
import torch

from oracle import native, restate
from oracle.restate import parity_gate
from paper_2405_16883_b200 import ops

pytestmark = pytest.mark.gpu

TOL = 1e-5


def make_csr(rng, m, n, lens):
    lens = np.asarray(lens, dtype=np.int64)
    lens = np.minimum(lens, n)
    rp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    ci = np.concatenate([np.sort(rng.choice(n, int(L), replace=False)) for L in lens]) if m else np.zeros(0)
    v = rng.uniform(-1, 1, rp[-1]).astype(np.float32)
    return rp, ci.astype(np.int64), v


def dev(rp, ci, v):
    return (torch.from_numpy(rp).int().cuda(), torch.from_numpy(ci).int().cuda(),
            torch.from_numpy(v).float().cuda())


STRUCTS = {
    "uniform": lambda r: (300, 200, r.integers(0, 30, 300)),
    "skewed": lambda r: (400, 500, np.where(np.arange(400) % 97 == 3, 450, r.integers(0, 4, 400))),
    "one_heavy": lambda r: (5, 6000, [0, 5999, 1, 0, 2]),
    "empty_rows": lambda r: (64, 50, np.where(np.arange(64) % 3 == 0, 0, 5)),
    "all_empty": lambda r: (17, 9, np.zeros(17, dtype=np.int64)),
    "single_row": lambda r: (1, 100, [37]),
    "trailing_empty": lambda r: (40, 30, np.where(np.arange(40) > 20, 0, 7)),
    # full rows: a COLTILE warp's chunk list (8 rows x 64 entries) overflows its shared-memory
    # stage, so the entries stream from global memory (coltile.cuh, `total > CTT_ECAP`)
    "dense_rows": lambda r: (200, 300, np.full(200, 300)),
}


@pytest.mark.parametrize("struct", list(STRUCTS))
@pytest.mark.parametrize("variant", ["row", "merge", "coltile"])
@pytest.mark.parametrize("k", [1, 3, 4, 13, 64, 128, 136, 260])
def test_spmm_variants(struct, variant, k):
    if variant == "coltile" and k % 4:
        pytest.skip("coltile needs k % 4 == 0")
    rng = np.random.default_rng(hash((struct, k)) % 2**32)
    m, n, lens = STRUCTS[struct](rng)
    rp, ci, v = make_csr(rng, m, n, lens)
    B = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    want = native.spmm_csr(rp, ci, v, B)
    bound = native.spmm_csr(rp, ci, np.abs(v), np.abs(B))
    R, Cc, V = dev(rp, ci, v)
    got = ops.spmm_csr(R, Cc, V, torch.from_numpy(B).cuda(), variant=variant).cpu().numpy()
    ok, worst = parity_gate(got, want, bound, TOL)
    assert ok, worst


@pytest.mark.parametrize("ipg", [1, 2, 7, 33, 128, 1000])
@pytest.mark.parametrize("k", [4, 64, 128])
def test_merge_carries_at_every_granularity(ipg, k):
    rng = np.random.default_rng(ipg * 100 + k)
    lens = np.concatenate([[0, 0], rng.integers(0, 6, 200), [3000], rng.integers(0, 3, 100), [0, 800, 0]])
    m = len(lens)
    rp, ci, v = make_csr(rng, m, 4000, lens)
    B = rng.uniform(-1, 1, (4000, k)).astype(np.float32)
    D = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    R, Cc, V = dev(rp, ci, v)
    part = ops.merge_partition(R, len(v), ipg)
    for relu in (False, True):
        got = ops.spmm_csr(R, Cc, V, torch.from_numpy(B).cuda(), addend=torch.from_numpy(D).cuda(),
                           relu=relu, variant="merge", partition=part).cpu().numpy()
        want = native.spmm_csr(rp, ci, v, B, addend=D, relu=relu)
        bound = native.spmm_csr(rp, ci, np.abs(v), np.abs(B), addend=np.abs(D))
        ok, worst = parity_gate(got, want, bound, TOL)
        assert ok, (relu, worst)


def test_merge_partition_matches_host_search():
    rng = np.random.default_rng(3)
    rp, ci, v = make_csr(rng, 500, 100, rng.integers(0, 12, 500))
    R, _, _ = dev(rp, ci, v)
    for ipg in (1, 5, 64):
        part = ops.merge_partition(R, len(v), ipg)
        st = part.starts.cpu().numpy().reshape(-1, 2)
        m, nnz = 500, len(v)
        # items: an entry weighs 1, a row end W (segreduce.cuh kRowCost); a group owns the
        # items that start in [g*ipg, (g+1)*ipg): entry q of row r starts at q + W*r, the
        # end of row r at rp[r+1] + W*r
        W = 2
        diags = np.minimum(np.arange(part.n_groups + 1) * ipg, W * m + nnz)
        end_starts = rp[1:] + W * np.arange(m)
        rows = np.searchsorted(end_starts, diags, side="left")     # row ends starting before diag
        pos = np.clip(diags - W * rows, rp[rows], rp[np.minimum(rows + 1, m)])
        assert part.n_groups == -(-(W * m + nnz) // ipg)
        assert np.array_equal(st[:, 0], rows)
        assert np.array_equal(st[:, 1], pos)


def test_spmm_deterministic_bitwise():
    rng = np.random.default_rng(11)
    lens = np.where(np.arange(2000) % 500 == 1, 20000, rng.integers(0, 10, 2000))
    rp, ci, v = make_csr(rng, 2000, 30000, lens)
    B = torch.randn(30000, 128, device="cuda")
    R, Cc, V = dev(rp, ci, v)
    a = ops.spmm_csr(R, Cc, V, B, variant="merge")
    b = ops.spmm_csr(R, Cc, V, B, variant="merge")
    assert torch.equal(a, b)


def test_strided_and_unaligned_operands():
    rng = np.random.default_rng(12)
    rp, ci, v = make_csr(rng, 100, 80, rng.integers(0, 10, 100))
    R, Cc, V = dev(rp, ci, v)
    big = torch.randn(80, 70, device="cuda")
    B = big[:, 1:38]  # row stride 70, unaligned start -> scalar path
    want = native.spmm_csr(rp, ci, v, B.cpu().numpy())
    bound = native.spmm_csr(rp, ci, np.abs(v), np.abs(B.cpu().numpy()))
    for variant in ("row", "merge"):
        got = ops.spmm_csr(R, Cc, V, B, variant=variant).cpu().numpy()
        assert parity_gate(got, want, bound, TOL)[0]


def test_batched_spmm():
    rng = np.random.default_rng(13)
    rp, ci, v = make_csr(rng, 300, 300, rng.integers(0, 40, 300))
    Z = 3
    vals = rng.uniform(0, 1, (Z, len(v))).astype(np.float32)
    B = rng.standard_normal((Z, 300, 64)).astype(np.float32)
    R, Cc, _ = dev(rp, ci, v)
    for variant in ("row", "merge"):
        got = ops.spmm_csr_batched(R, Cc, torch.from_numpy(vals).cuda(), torch.from_numpy(B).cuda(),
                                   variant=variant).cpu().numpy()
        for z in range(Z):
            want = native.spmm_csr(rp, ci, vals[z], B[z])
            bound = native.spmm_csr(rp, ci, vals[z], np.abs(B[z]))
            assert parity_gate(got[z], want, bound, TOL)[0]


@pytest.mark.parametrize("d", [4, 8, 16, 32, 64, 128])
@pytest.mark.parametrize("heads", [1, 3])
def test_sddmm(d, heads):
    rng = np.random.default_rng(d * 10 + heads)
    rp, ci, mv = make_csr(rng, 120, 90, rng.integers(0, 50, 120))
    Q = rng.standard_normal((heads, 120, d)).astype(np.float32)
    K = rng.standard_normal((heads, 90, d)).astype(np.float32)
    R, Cc, MV = dev(rp, ci, mv)
    got = ops.sddmm_csr(R, Cc, torch.from_numpy(Q).cuda(), torch.from_numpy(K).cuda(), maskvals=MV,
                        scale=0.5).cpu().numpy()
    for h in range(heads):
        want = 0.5 * native.sddmm_csr(rp, ci, mv, Q[h], K[h])
        bound = 0.5 * native.sddmm_csr(rp, ci, np.abs(mv), np.abs(Q[h]), np.abs(K[h]))
        rows = np.repeat(np.arange(120), np.diff(rp))
        err = np.abs(got[h] - want)
        lim = np.zeros(120)
        np.maximum.at(lim, rows, bound)
        assert np.all(err <= TOL * lim[rows] + 0.0)


def test_softmax_and_fused_attention():
    rng = np.random.default_rng(21)
    m = n = 200
    lens = np.minimum(np.arange(m) + 1, 40)
    rp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    ci = np.concatenate([np.arange(max(0, q - L + 1), q + 1) for q, L in zip(range(m), lens)])
    mv = np.ones(len(ci), dtype=np.float32)
    H, d = 2, 64
    Q = rng.standard_normal((H, m, d)).astype(np.float32)
    K = rng.standard_normal((H, n, d)).astype(np.float32)
    V = rng.standard_normal((H, n, d)).astype(np.float32)
    R, Cc, MV = dev(rp, ci, mv)
    Qt, Kt, Vt = (torch.from_numpy(x).cuda() for x in (Q, K, V))
    O, S, P = ops.sparse_attention(R, Cc, Qt, Kt, Vt, maskvals=MV, scale=0.125, return_probs=True)
    O2 = ops.sparse_attention(R, Cc, Qt, Kt, Vt, maskvals=MV, scale=0.125)
    S_u = ops.sddmm_csr(R, Cc, Qt, Kt, maskvals=MV, scale=0.125)
    P_u = ops.segment_softmax_(R, S_u.clone())
    O_u = ops.spmm_csr_batched(R, Cc, P_u.contiguous(), Vt)
    for h in range(H):
        s_ref = 0.125 * native.sddmm_csr(rp, ci, mv, Q[h], K[h])
        p_ref = native.segment_softmax(rp, s_ref)
        o_ref = native.spmm_csr(rp, ci, p_ref, V[h])
        o_bound = native.spmm_csr(rp, ci, p_ref, np.abs(V[h]))
        s_bound = 0.125 * native.sddmm_csr(rp, ci, mv, np.abs(Q[h]), np.abs(K[h]))
        assert np.all(np.abs(S[h].cpu().numpy() - s_ref) <= TOL * s_bound + 1e-12)
        assert np.abs(P[h].cpu().numpy() - p_ref).max() <= TOL
        assert np.abs(P_u[h].cpu().numpy() - p_ref).max() <= TOL
        for o in (O[h], O2[h], O_u[h]):
            assert parity_gate(o.cpu().numpy(), o_ref, o_bound, TOL)[0]


def test_coo_segments_and_mttkrp():
    rng = np.random.default_rng(31)
    dim = 300
    i = np.sort(np.minimum(rng.zipf(1.3, 5000) - 1, dim - 1))
    j = rng.integers(0, dim, 5000)
    k = rng.integers(0, dim, 5000)
    key = np.unique((i * dim + j) * dim + k)
    i, j, k = key // (dim * dim), (key // dim) % dim, key % dim
    vals = rng.uniform(0, 1, len(key)).astype(np.float32)
    B = rng.uniform(0, 1, (dim, 32)).astype(np.float32)
    C = rng.uniform(0, 1, (dim, 32)).astype(np.float32)
    seg = ops.coo_segments(torch.from_numpy(i).int().cuda())
    rows_ref, ptr_ref = restate.coo_segments(i)
    assert np.array_equal(seg.rows.cpu().numpy(), rows_ref)
    assert np.array_equal(seg.ptr.cpu().numpy(), ptr_ref)
    Jt, Kt = torch.from_numpy(j).int().cuda(), torch.from_numpy(k).int().cuda()
    Vt = torch.from_numpy(vals).cuda()
    want = native.mttkrp(ptr_ref, j, k, vals, B, C)
    for variant in ("row", "merge"):
        for R in (32, 7):
            got = ops.mttkrp_coo3(seg, Jt, Kt, Vt, torch.from_numpy(B[:, :R].copy()).cuda(),
                                  torch.from_numpy(C[:, :R].copy()).cuda(), variant=variant).cpu().numpy()
            assert parity_gate(got, want[:, :R], want[:, :R], TOL)[0]


def _zipf_coo3(seed, dim, draws):
    rng = np.random.default_rng(seed)
    i = np.minimum(rng.zipf(1.3, draws) - 1, dim - 1)
    j = np.minimum(rng.zipf(1.2, draws) - 1, dim - 1)
    k = rng.integers(0, dim, draws)
    key = np.unique((i * dim + j) * dim + k)
    i, j, k = key // (dim * dim), (key // dim) % dim, key % dim
    vals = rng.uniform(0, 1, len(key)).astype(np.float32)
    return rng, i, j, k, vals


@pytest.mark.parametrize("R", [4, 7, 32, 64, 128])
@pytest.mark.parametrize("ipg", [None, 1, 2, 3, 9, 33, 250, 1000])
def test_mttkrp_prepared_items_matches_raw_kernel_and_oracle(R, ipg):
    """The cp.async-staged kernel over prepared items (stc_mttkrp_coo3_prepared_f32): bit-identical
    to the raw-stream merge kernel on the same partition, and within the gate of the oracle — at
    every group size (carries inside and across CTAs, groups that start mid-fiber, empty groups)."""
    dim = 400
    rng, i, j, k, vals = _zipf_coo3(77 + R, dim, 30000)
    B = rng.uniform(-1, 1, (dim, R)).astype(np.float32)
    C = rng.uniform(-1, 1, (dim, R)).astype(np.float32)
    seg = ops.coo_segments(torch.from_numpy(i).int().cuda())
    _, ptr_ref = restate.coo_segments(i)
    Jt, Kt, Vt = torch.from_numpy(j).int().cuda(), torch.from_numpy(k).int().cuda(), torch.from_numpy(vals).cuda()
    Bt, Ct = torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda()
    fkey = (dim, Bt.stride(0), dim, Ct.stride(0))
    prep = ops.merge_partition(seg.ptr, len(vals), ipg, k=R, kind="mttkrp", jcrd=Jt, kcrd=Kt, vals=Vt, factors=fkey)
    assert prep.items is not None and prep.items.numel() == 16 * len(vals)
    raw = ops.merge_partition(seg.ptr, len(vals), prep.items_per_group, k=R, kind="mttkrp")
    assert raw.items is None
    got = ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=prep)
    ref = ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=raw)
    assert torch.equal(got, ref)
    for _ in range(3):  # arrival counters back at zero: relaunches are bit-stable
        assert torch.equal(ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=prep), got)
    want = native.mttkrp(ptr_ref, j, k, vals, B, C)
    bound = native.mttkrp(ptr_ref, j, k, vals, np.abs(B), np.abs(C))
    assert parity_gate(got.cpu().numpy(), want, bound, TOL)[0]


def test_mttkrp_prepared_plan_is_bound_to_its_buffers_and_factor_shapes():
    dim, R = 50, 32
    rng, i, j, k, vals = _zipf_coo3(5, dim, 2000)
    seg = ops.coo_segments(torch.from_numpy(i).int().cuda())
    Jt, Kt, Vt = torch.from_numpy(j).int().cuda(), torch.from_numpy(k).int().cuda(), torch.from_numpy(vals).cuda()
    Bt = torch.from_numpy(rng.uniform(0, 1, (dim, R)).astype(np.float32)).cuda()
    Ct = torch.from_numpy(rng.uniform(0, 1, (dim, R)).astype(np.float32)).cuda()
    part = ops.merge_partition(seg.ptr, len(vals), k=R, kind="mttkrp", jcrd=Jt, kcrd=Kt, vals=Vt,
                               factors=(dim, R, dim, R))
    M0 = ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=part)
    # default call (no plan given) prepares the same way
    assert torch.equal(ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct), M0)
    wide = torch.zeros((dim, 2 * R), device="cuda")
    wide[:, :R] = Bt
    with pytest.raises(ValueError, match="prepared for factors"):
        ops.mttkrp_coo3(seg, Jt, Kt, Vt, wide[:, :R], Ct, partition=part)   # ldb = 64: other offsets
    with pytest.raises(ValueError, match="prepared items of other"):
        ops.mttkrp_coo3(seg, Jt, Kt, Vt.clone(), Bt, Ct, partition=part)
    Vt.mul_(2.0)                                                              # values modified in place
    with pytest.raises(ValueError, match="prepared items of other"):
        ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=part)
    # strided factor: a fresh plan for its leading dimension
    got = ops.mttkrp_coo3(seg, Jt, Kt, Vt, wide[:, :R], Ct)
    assert torch.allclose(got, 2.0 * M0, rtol=1e-6, atol=0)


@pytest.mark.parametrize("seq,window,nrand,heads", [(200, 40, 8, 2), (700, 256, 64, 1), (130, 300, 5, 3)])
def test_tiled_attention_matches_oracle(seq, window, nrand, heads):
    from paper_2405_16883_b200 import synthetic

    M, Q, K, V = synthetic.cfg4(seq=seq, heads=heads, dim=64, window=window, n_random=nrand)
    rng = np.random.default_rng(seq)
    mv = np.where(rng.random(M.nnz) < 0.1, 0.0, rng.uniform(0.5, 2.0, M.nnz)).astype(np.float32)  # incl. zeros
    R, Cc, MV = dev(M.rowptr, M.colidx, mv)
    plan = ops.attention_tile_plan(R, Cc, MV, seq)
    assert plan is not None and plan.dense_share > 0.3
    Qt, Kt, Vt = (torch.from_numpy(x).cuda() for x in (Q, K, V))
    O = ops.sparse_attention_tiled(plan, Qt, Kt, Vt, scale=0.125).cpu().numpy()
    for h in range(heads):
        s = 0.125 * native.sddmm_csr(M.rowptr, M.colidx, mv, Q[h], K[h])
        p = native.segment_softmax(M.rowptr, s)
        o = native.spmm_csr(M.rowptr, M.colidx, p, V[h])
        ob = native.spmm_csr(M.rowptr, M.colidx, p, np.abs(V[h]))
        ok, worst = parity_gate(O[h], o, ob, TOL)
        assert ok, worst


# ---- dense operands of 2^32 elements or more (64-bit gathers, spmm_wide.cu) -------------------------

def _wide_operand(n, k, used, rng):
    """An (n, k) fp32 device operand (> 2^32 elements, ~17 GB) whose rows in `used` hold
    seeded values; the other rows are never read. Returns (B, compact host copy, remap)."""
    B = torch.empty((n, k), dtype=torch.float32, device="cuda")
    used = np.unique(used)
    vals = rng.uniform(-1, 1, (len(used), k)).astype(np.float32)
    B[torch.from_numpy(used).cuda().long()] = torch.from_numpy(vals).cuda()
    remap = np.full(n, -1, dtype=np.int64)
    remap[used] = np.arange(len(used))
    return B, vals, remap


@pytest.mark.parametrize("variant", ["row", "merge"])
def test_spmm_dense_operand_beyond_32bit_offsets(variant):
    rng = np.random.default_rng(77)
    k = 128
    n = (1 << 32) // k + 4099                     # (n + 1) * k > 2^32: 64-bit gathers
    m = 700
    # rows: ~half their columns near the start, the rest past the 32-bit offset boundary
    rows = []
    for L in np.where(np.arange(m) % 50 == 7, 900, rng.integers(0, 24, m)):
        c = np.unique(np.concatenate([rng.integers(0, 1000, L // 2 + 1), rng.integers(n - 200_000, n, L)]))[:L]
        rows.append(np.sort(c))
    rp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum([len(r) for r in rows], out=rp[1:])
    ci = np.concatenate(rows).astype(np.int64)
    v = rng.uniform(-1, 1, len(ci)).astype(np.float32)
    try:
        B, host_rows, remap = _wide_operand(n, k, ci, rng)
    except torch.OutOfMemoryError:
        pytest.skip("device too small for a 2^32-element operand")
    R, C, V = dev(rp, ci, v)
    got = ops.spmm_csr(R, C, V, B, relu=True, variant=variant).cpu().numpy()
    want = native.spmm_csr(rp, remap[ci], v, host_rows, relu=True)
    bound = native.spmm_csr(rp, remap[ci], np.abs(v), np.abs(host_rows))
    assert parity_gate(got, want, bound, TOL)[0]
    del B
    torch.cuda.empty_cache()


def test_mttkrp_factor_beyond_32bit_offsets():
    rng = np.random.default_rng(78)
    R = 32
    nj = (1 << 32) // R + 777                    # B has more than 2^32 elements
    dim_i, dim_k = 200, 300
    i = np.sort(rng.integers(0, dim_i, 4000))
    j = np.where(rng.random(4000) < 0.5, rng.integers(0, 500, 4000), rng.integers(nj - 5000, nj, 4000))
    k = rng.integers(0, dim_k, 4000)
    key = np.unique(np.stack([i, j, k], 1), axis=0)
    i, j, k = key[:, 0], key[:, 1], key[:, 2]
    vals = rng.uniform(0, 1, len(i)).astype(np.float32)
    try:
        B, host_b, remap = _wide_operand(nj, R, j, rng)
    except torch.OutOfMemoryError:
        pytest.skip("device too small for a 2^32-element operand")
    Cf = rng.uniform(0, 1, (dim_k, R)).astype(np.float32)
    seg = ops.coo_segments(torch.from_numpy(i).int().cuda())
    _, ptr_ref = restate.coo_segments(i)
    Jt, Kt = torch.from_numpy(j).int().cuda(), torch.from_numpy(k).int().cuda()
    Vt = torch.from_numpy(vals).cuda()
    want = native.mttkrp(ptr_ref, remap[j], k, vals, host_b, Cf)
    bound = native.mttkrp(ptr_ref, remap[j], k, np.abs(vals), np.abs(host_b), np.abs(Cf))
    for variant in ("row", "merge"):
        got = ops.mttkrp_coo3(seg, Jt, Kt, Vt, B, torch.from_numpy(Cf).cuda(), variant=variant).cpu().numpy()
        assert parity_gate(got, want, bound, TOL)[0]
    del B
    torch.cuda.empty_cache()


def test_interleave_long_rows_kernel():
    """stc_merge_interleave: rows longer than the span become G interleaved sequences
    (entries 0, G, 2G, ..., 1, G+1, ...); shorter rows are copied unchanged."""
    rng = np.random.default_rng(0)
    lens = np.array([3, 1200, 0, 64, 65, 2000, 7, 0, 129])
    rp = np.concatenate([[0], np.cumsum(lens)])
    ci = rng.integers(0, 10**6, rp[-1]).astype(np.int64)
    va = rng.random(rp[-1]).astype(np.float32)
    c, v = ops.interleave_long_rows(*dev(rp, ci, va), 64)
    c, v = c.cpu().numpy(), v.cpu().numpy()
    for r in range(len(lens)):
        a, b = rp[r], rp[r + 1]
        order = np.arange(b - a)
        if b - a > 64:
            g = -(-(b - a) // 64)
            order = np.concatenate([np.arange(j, b - a, g) for j in range(g)])
        assert np.array_equal(c[a:b], ci[a:b][order]) and np.array_equal(v[a:b], va[a:b][order])


def test_merge_with_interleaved_plan_matches_oracle():
    rng = np.random.default_rng(5)
    m, n, k = 400, 3000, 128
    lens = np.where(np.arange(m) % 37 == 0, rng.integers(1500, 2900, m), rng.integers(0, 12, m))
    rp, ci, v = make_csr(rng, m, n, lens)
    R, C, V = dev(rp, ci, v)
    B = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    part = ops.merge_partition(R, len(v), 64, k=k, colidx=C, vals=V)
    assert part.colidx is not None
    Bt = torch.from_numpy(B).cuda()
    got = ops.spmm_csr(R, C, V, Bt, variant="merge", partition=part).cpu().numpy()
    again = ops.spmm_csr(R, C, V, Bt, variant="merge", partition=part).cpu().numpy()
    assert np.array_equal(got, again)  # fixed order: bit-reproducible
    want = native.spmm_csr(rp, ci, v, B)
    assert parity_gate(got, want, native.spmm_csr(rp, ci, np.abs(v), np.abs(B)), TOL)[0]


# ---- non-finite values in operand rows no stored entry references ---------------

def test_coltile_padding_ignores_nonfinite_unreferenced_rows():
    """COLTILE pads each row's entries per 64-column chunk to a multiple of 4; the padding must
    contribute nothing even when a B row of that chunk that the row never references holds
    Inf / NaN (the reference multiplies stored entries only)."""
    rng = np.random.default_rng(41)
    m, n, k = 256, 256, 128
    lens = rng.integers(1, 7, m)                      # rows need padding in most chunks
    rp, ci, v = make_csr(rng, m, n, lens)
    B = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    used = np.zeros(n, bool)
    used[ci] = True
    bad = np.flatnonzero(~used)
    assert bad.size > 0
    B[bad[0::2]] = np.inf
    B[bad[1::2]] = np.nan
    R, C, V = dev(rp, ci, v)
    for variant in ("coltile", "merge", "row"):
        got = ops.spmm_csr(R, C, V, torch.from_numpy(B).cuda(), variant=variant).cpu().numpy()
        assert np.isfinite(got).all(), variant
        want = native.spmm_csr(rp, ci, v, np.nan_to_num(B, nan=0, posinf=0))
        bound = native.spmm_csr(rp, ci, np.abs(v), np.abs(np.nan_to_num(B, nan=0, posinf=0)))
        assert parity_gate(got, want, bound, TOL)[0], variant
    # a referenced Inf still propagates like the reference (w * Inf, or 0 * Inf = NaN)
    B2 = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    B2[ci[0]] = np.inf
    got = ops.spmm_csr(R, C, V, torch.from_numpy(B2).cuda(), variant="coltile").cpu().numpy()
    want = native.spmm_csr(rp, ci, v, B2)
    assert np.array_equal(np.isnan(got), np.isnan(want)) and np.array_equal(np.isinf(got), np.isinf(want))


@pytest.mark.parametrize("shape", [(300, 200, 128), (130, 1000, 260), (128, 63, 4), (64, 127, 132)])
def test_coltile_operand_paths_agree(shape, monkeypatch):
    """The COLTILE producer stages B by one tiled TMA copy per 63-row chunk (tensor map, zero fill
    past n and k) or, when the operand cannot be mapped, by one bulk copy per row: both must give
    the same bits (same plan, same summation order), ragged edges included."""
    m, n, k = shape
    rng = np.random.default_rng(m * 7 + n)
    rp, ci, v = make_csr(rng, m, n, rng.integers(0, min(n, 40), m))
    B = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    R, C, V = dev(rp, ci, v)
    Bt = torch.from_numpy(B).cuda()
    tiled = ops.spmm_csr(R, C, V, Bt, variant="coltile")
    monkeypatch.setenv("STC_COLTILE_ROW_COPIES", "1")
    by_row = ops.spmm_csr(R, C, V, Bt, variant="coltile")
    monkeypatch.delenv("STC_COLTILE_ROW_COPIES")
    assert torch.equal(tiled, by_row)
    want = native.spmm_csr(rp, ci, v, B)
    bound = native.spmm_csr(rp, ci, np.abs(v), np.abs(B))
    assert parity_gate(tiled.cpu().numpy(), want, bound, TOL)[0]
    # a column slice of a wider operand: pitch != width, base offset by 4 floats
    wide = torch.from_numpy(rng.uniform(-1, 1, (n, k + 8)).astype(np.float32)).cuda()
    view = wide[:, 4:4 + k]
    got = ops.spmm_csr(R, C, V, view, variant="coltile")
    assert torch.equal(got, ops.spmm_csr(R, C, V, view.contiguous(), variant="coltile"))


def test_tiled_attention_ignores_nonfinite_unreferenced_value_rows():
    """Dense 64x64 tiles hold absent slots; a V row that some rows of the block do not
    reference may be Inf / NaN without touching those rows (rows that reference it do)."""
    from paper_2405_16883_b200 import synthetic

    M, Q, K, V = synthetic.cfg4(seq=256, heads=1, dim=64, window=48, n_random=4)
    R, Cc, MV = dev(M.rowptr, M.colidx, M.vals)
    plan = ops.attention_tile_plan(R, Cc, MV, 256)
    assert plan is not None
    bad = 100
    V = V.copy()
    V[0, bad] = np.inf
    Qt, Kt, Vt = (torch.from_numpy(x).cuda() for x in (Q, K, V))
    O = ops.sparse_attention_tiled(plan, Qt, Kt, Vt, scale=0.125).cpu().numpy()[0]
    refs = np.zeros(M.shape[0], bool)
    rows = np.repeat(np.arange(M.shape[0]), np.diff(M.rowptr))
    refs[rows[M.colidx == bad]] = True
    assert np.isfinite(O[~refs]).all()
    s = 0.125 * native.sddmm_csr(M.rowptr, M.colidx, M.vals, Q[0], K[0])
    p = native.segment_softmax(M.rowptr, s)
    o = native.spmm_csr(M.rowptr, M.colidx, p, V[0])
    ob = native.spmm_csr(M.rowptr, M.colidx, p, np.abs(np.nan_to_num(V[0], posinf=0)))
    keep = ~refs
    assert parity_gate(O[keep], o[keep], ob[keep], TOL)[0]
    assert np.array_equal(np.isfinite(O[refs]), np.isfinite(o[refs]))


# ---- cross-CTA carry protocol under repetition ------------------------------------------------

@pytest.mark.parametrize("ipg", [1, 2, 5])
def test_merge_carries_bitwise_stable_over_many_launches(ipg):
    """Rows cut across many CTAs (items per group 1..5): the last-arriving CTA combines the
    carries in position order. 300 back-to-back launches (different CTA arrival orders) must
    all be bit-identical and match the oracle; the arrival counters must return to zero."""
    rng = np.random.default_rng(ipg)
    lens = np.where(np.arange(64) % 9 == 0, 700, rng.integers(0, 5, 64))
    rp, ci, v = make_csr(rng, 64, 800, lens)
    R, C, V = dev(rp, ci, v)
    B = torch.randn(800, 64, device="cuda")
    part = ops.merge_partition(R, len(v), ipg)
    ws = ops.spmm_workspace(64, len(v), 64, "merge", part.items_per_group, 1, "cuda")
    first = ops.spmm_csr(R, C, V, B, variant="merge", partition=part, workspace=ws, relu=True)
    outs = [ops.spmm_csr(R, C, V, B, variant="merge", partition=part, workspace=ws, relu=True) for _ in range(300)]
    torch.cuda.synchronize()
    assert all(torch.equal(first, o) for o in outs)
    # workspace = head partials | tail partials (n_cta x 64 floats each) | n_cta arrival counters
    n_cta = -(-part.n_groups // 16)  # k = 64: 16-lane groups, 16 per CTA
    counters = ws.view(torch.int32)[2 * n_cta * 64: 2 * n_cta * 64 + n_cta]
    assert int(counters.abs().sum()) == 0
    want = native.spmm_csr(rp, ci, v, B.cpu().numpy().astype(np.float64), relu=True)
    bound = native.spmm_csr(rp, ci, np.abs(v), np.abs(B.cpu().numpy().astype(np.float64)))
    assert parity_gate(first.cpu().numpy(), want, bound, TOL)[0]


# ---- COLTILE stage / TMEM-buffer hand-offs under repetition -----------------------------------

def test_coltile_pipeline_bitwise_stable_over_many_launches():
    """COLTILE hands B chunks from the TMA stage ring to the four fill warps and on to the 28
    consumer warps through mbarriers (stage landed / stage copied, TMEM buffer written / read, per
    lane quarter). A missed wait shows up as a stale or half-written chunk: 40 chunks per CTA
    (n = 2500), unequal work per warp (row lengths 0..300), two column tiles with a ragged edge
    (k = 132), 100 back-to-back launches -- all outputs must be bit-identical and equal to the
    oracle, with an addend + ReLU epilogue as well."""
    rng = np.random.default_rng(77)
    m, n, k = 500, 2500, 132
    lens = np.where(np.arange(m) % 7 == 0, 300, rng.integers(0, 40, m))
    rp, ci, v = make_csr(rng, m, n, lens)
    B = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    D = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    R, C, V = dev(rp, ci, v)
    Bt, Dt = torch.from_numpy(B).cuda(), torch.from_numpy(D).cuda()
    plan = ops.coltile_plan(R, C, n, V)
    first = ops.spmm_csr(R, C, V, Bt, addend=Dt, relu=True, variant="coltile", partition=plan)
    outs = [ops.spmm_csr(R, C, V, Bt, addend=Dt, relu=True, variant="coltile", partition=plan) for _ in range(100)]
    torch.cuda.synchronize()
    assert all(torch.equal(first, o) for o in outs)
    want = native.spmm_csr(rp, ci, v, B, addend=D, relu=True)
    bound = native.spmm_csr(rp, ci, np.abs(v), np.abs(B), addend=np.abs(D))
    assert parity_gate(first.cpu().numpy(), want, bound, TOL)[0]


def test_coltile_plan_rejects_another_matrix():
    """A COLTILE plan encodes one matrix (structure and values): using it with another m / n /
    nnz, other buffers, or values modified in place must raise instead of computing with stale
    entries or indexing the plan out of range."""
    rng = np.random.default_rng(5)
    rp, ci, v = make_csr(rng, 300, 200, rng.integers(0, 30, 300))
    R, C, V = dev(rp, ci, v)
    B = torch.randn(200, 128, device="cuda")
    plan = ops.coltile_plan(R, C, 200, V)
    ops.spmm_csr(R, C, V, B, variant="coltile", partition=plan)
    with pytest.raises(ValueError):
        ops.spmm_csr(R, C, V.clone(), B, variant="coltile", partition=plan)      # other value buffer
    with pytest.raises(ValueError):
        ops.spmm_csr(R, C, V, torch.randn(264, 128, device="cuda"), variant="coltile", partition=plan)  # other n
    V.mul_(2.0)                                                                   # values changed in place
    with pytest.raises(ValueError):
        ops.spmm_csr(R, C, V, B, variant="coltile", partition=plan)


@pytest.mark.parametrize("seed", range(24))
def test_coltile_random_shapes(seed):
    """COLTILE forced on random shapes around its block edges (224-row blocks, 63-row operand
    chunks, 128-column tiles): ragged last block / chunk / tile, empty rows, rows denser than the
    staged list, addend and ReLU epilogues -- against the float64 oracle."""
    rng = np.random.default_rng(9000 + seed)
    m = int(rng.choice([1, 7, 223, 224, 225, 449, int(rng.integers(1, 700))]))
    n = int(rng.choice([1, 62, 63, 64, 126, 127, int(rng.integers(1, 400))]))
    k = 4 * int(rng.choice([1, 31, 32, 33, 64, int(rng.integers(1, 70))]))
    dens = float(rng.choice([0.0, 0.02, 0.3, 1.0]))
    lens = rng.binomial(n, dens, m)
    lens[rng.random(m) < 0.2] = 0
    rp, ci, v = make_csr(rng, m, n, lens)
    B = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    D = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    R, C, V = dev(rp, ci, v)
    relu = bool(seed & 1)
    use_d = bool(seed & 2)
    got = ops.spmm_csr(R, C, V, torch.from_numpy(B).cuda(), variant="coltile", relu=relu,
                       addend=torch.from_numpy(D).cuda() if use_d else None).cpu().numpy()
    want = native.spmm_csr(rp, ci, v, B, addend=D if use_d else None, relu=relu)
    bound = native.spmm_csr(rp, ci, np.abs(v), np.abs(B), addend=np.abs(D) if use_d else None)
    ok, worst = parity_gate(got, want, bound, TOL)
    assert ok, (m, n, k, dens, worst)
