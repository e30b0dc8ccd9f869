"""Small instances of every kernel in libstc.so, for compute-sanitizer runs:

  compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
  compute-sanitizer --tool racecheck python tools/sanitize_cases.py
  compute-sanitizer --tool synccheck python tools/sanitize_cases.py
  compute-sanitizer --tool initcheck python tools/sanitize_cases.py

Covers: merge_kernel (items per group 1 / 3 / 37 so rows are cut inside and across CTAs,
ReLU and dense-addend fix-ups, interleaved long rows, batched, MTTKRP, 64-bit-offset ops
not included: 17 GB operands), row_kernel, coltile_tmem_kernel (+ plan kernels, a chunk
list that overflows the shared-memory stage), sddmm_kernel, segsoftmax_kernel,
attention_kernel, attn_tile8_kernel + remainder, merge_partition / interleave /
coo_segments plan kernels, SpGEMM dense-window and expand-sort-compress paths, element-wise
union / intersection. Results are checked against torch float64 on the same inputs so a
sanitizer run that silently changes numbers also fails.
"""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402

rng = np.random.default_rng(11)
dev = "cuda"


def csr(m, n, lens):
    lens = np.minimum(np.asarray(lens, dtype=np.int64), n)
    rp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    ci = np.concatenate([np.sort(rng.choice(n, int(L), replace=False)) for L in lens])
    v = rng.uniform(-1, 1, rp[-1]).astype(np.float32)
    return (torch.from_numpy(rp).int().to(dev), torch.from_numpy(ci).int().to(dev), torch.from_numpy(v).to(dev))


def dense_of(R, C, V, m, n):
    A = torch.zeros(m, n, dtype=torch.float64, device=dev)
    rows = torch.repeat_interleave(torch.arange(m, device=dev), (R[1:] - R[:-1]).long())
    A[rows, C.long()] = V.double()
    return A


def close(got, want, what):
    err = (got.double() - want).abs().max().item() if got.numel() else 0.0
    scale = max(want.abs().max().item(), 1.0) if want.numel() else 1.0
    assert err <= 1e-4 * scale, f"{what}: max err {err}"


# ---- SpMM: ROW / MERGE (several granularities, epilogues) / COLTILE -----------------------
m, n = 300, 500
lens = np.where(np.arange(m) % 97 == 3, 480, rng.integers(0, 6, m))
R, C, V = csr(m, n, lens)
Ad = dense_of(R, C, V, m, n)
for k in (4, 13, 128, 136):
    B = torch.randn(n, k, device=dev)
    D = torch.randn(m, k, device=dev)
    want = Ad @ B.double()
    close(ops.spmm_csr(R, C, V, B, variant="row"), want, f"row k={k}")
    for ipg in (1, 3, 37):
        part = ops.merge_partition(R, V.numel(), ipg)
        got = ops.spmm_csr(R, C, V, B, variant="merge", partition=part, relu=True, addend=D)
        close(got, torch.clamp_min(want + D.double(), 0), f"merge k={k} ipg={ipg}")
    part = ops.merge_partition(R, V.numel(), 64, k=k, colidx=C, vals=V)  # interleaved long rows
    close(ops.spmm_csr(R, C, V, B, variant="merge", partition=part), want, f"merge interleaved k={k}")
    if k % 4 == 0:
        close(ops.spmm_csr(R, C, V, B, variant="coltile"), want, f"coltile k={k}")
Rd, Cd, Vd = csr(200, 300, np.full(200, 300))  # full rows: COLTILE entry lists overflow the stage
Bd = torch.randn(300, 128, device=dev)
close(ops.spmm_csr(Rd, Cd, Vd, Bd, variant="coltile"), dense_of(Rd, Cd, Vd, 200, 300) @ Bd.double(), "coltile dense")

# batched (head-batched PV shape)
Z = 3
vals = torch.rand(Z, V.numel(), device=dev)
Bz = torch.randn(Z, n, 16, device=dev)
got = ops.spmm_csr_batched(R, C, vals, Bz, variant="merge")
for z in range(Z):
    close(got[z], dense_of(R, C, vals[z], m, n) @ Bz[z].double(), f"batched z={z}")

# ---- SDDMM, softmax, fused attention (per-row), tiled attention --------------------------
M, Q, K, Vv = synthetic.cfg4(seq=200, heads=2, dim=64, window=40, n_random=8)
Rm, Cm, MV = (torch.from_numpy(M.rowptr).int().to(dev), torch.from_numpy(M.colidx).int().to(dev),
              torch.from_numpy(M.vals).to(dev))
Qt, Kt, Vt = (torch.from_numpy(x).to(dev) for x in (Q, K, Vv))
S = ops.sddmm_csr(Rm, Cm, Qt, Kt, maskvals=MV, scale=0.125)
P = ops.segment_softmax_(Rm, S.clone())
O, S2, P2 = ops.sparse_attention(Rm, Cm, Qt, Kt, Vt, maskvals=MV, scale=0.125, return_probs=True)
O_unf = ops.spmm_csr_batched(Rm, Cm, P.contiguous(), Vt)
close(O, O_unf.double(), "fused vs unfused attention")
plan = ops.attention_tile_plan(Rm, Cm, MV, 200)
O_t = ops.sparse_attention_tiled(plan, Qt, Kt, Vt, scale=0.125)
close(O_t, O_unf.double(), "tiled attention")
for d in (4, 16, 100):
    Qd, Kd = torch.randn(m, d, device=dev), torch.randn(n, d, device=dev)
    if d <= 64:
        ops.sddmm_csr(R, C, Qd, Kd, maskvals=V)

# ---- COO segmentation + MTTKRP --------------------------------------------------------------
dim = 120
i = np.sort(np.minimum(rng.zipf(1.3, 3000) - 1, dim - 1))
j, kk = rng.integers(0, dim, 3000), rng.integers(0, dim, 3000)
key = np.unique((i * dim + j) * dim + kk)
i, j, kk = key // (dim * dim), (key // dim) % dim, key % dim
tv = rng.uniform(0, 1, len(key)).astype(np.float32)
seg = ops.coo_segments(torch.from_numpy(i).int().to(dev))
Bf, Cf = torch.rand(dim, 32, device=dev), torch.rand(dim, 32, device=dev)
Jt, Kt3 = (torch.from_numpy(x).int().to(dev) for x in (j, kk))
Tv = torch.from_numpy(tv).to(dev)
want = torch.zeros(dim, 32, dtype=torch.float64, device=dev)
want.index_add_(0, torch.from_numpy(i).to(dev), Tv.double()[:, None] * Bf.double()[Jt.long()] * Cf.double()[Kt3.long()])
for variant in ("merge", "row"):
    got = ops.mttkrp_coo3(seg, Jt, Kt3, Tv, Bf, Cf, variant=variant)
    close(got, want[seg.rows.long()], f"mttkrp {variant}")

# ---- sparse x sparse -------------------------------------------------------------------------
A2 = csr(80, 90, rng.integers(0, 10, 80))
B2 = csr(90, 70, rng.integers(0, 10, 90))
r = ops.spgemm_csr(*A2, *B2, 70)
B3 = csr(90, 7000, rng.integers(0, 30, 90))  # > 6144 output columns: expand-sort-compress path
r3 = ops.spgemm_csr(*A2, *B3, 7000)
E1, E2 = csr(80, 90, rng.integers(0, 12, 80)), csr(80, 90, rng.integers(0, 12, 80))
for op in ("add", "mul"):
    ops.csr_ewise(op, *E1, *E2)
torch.cuda.synchronize()
print("sanitize_cases: all kernels ran, results match float64 torch")
