"""torch interception (§8(f)-2): sparse inferred outputs stay sparse, plans are cached per
operand signature, ``out=`` is honoured and unsupported calls raise instead of densifying.
Semantics: `/root/reference/PAPER.md:45, 96, 328-330, 430` (intercept torch calls on declared
sparse tensors; the output format is inferred)."""

import numpy as np
import pytest
import torch

import paper_2405_16883_b200 as st
from oracle import native
from oracle.restate import parity_gate
from paper_2405_16883_b200 import synthetic, torch_dispatch

from helpers import random_tensor

pytestmark = pytest.mark.gpu


def test_einsum_sddmm_returns_the_sparse_tensor():
    r = np.random.default_rng(3)
    M = random_tensor(r, (50, 40), "csr", 0.2, "M")
    Q = torch.randn(50, 16, device="cuda")
    K = torch.randn(40, 16, device="cuda")
    S = torch.einsum("ij,id,jd->ij", M, Q, K)
    assert isinstance(S, st.Tensor) and S.format.name() == "csr"
    L = M.storage.levels[1]
    assert torch.equal(S.storage.levels[1].pos, L.pos) and torch.equal(S.storage.levels[1].crd, L.crd)
    dense = torch.from_numpy(st.to_dense(M)).cuda().float() * (Q @ K.T)
    torch.testing.assert_close(st.to_torch(S), dense, rtol=1e-5, atol=1e-5)


def test_einsum_multihead_sddmm_at_cfg4_shape_stays_sparse():
    """torch.einsum("ij,hid,hjd->hij") on the cfg4 mask and 16 heads: the result is the
    [dense, dense, compressed] tensor (H * nnz values), never the 16 x 8192 x 8192 dense."""
    Mh, Q, K, _ = synthetic.cfg4()
    M = st.csr_from_arrays(Mh.rowptr, Mh.colidx, Mh.vals, Mh.shape, name="M")
    Qt, Kt = torch.from_numpy(Q).cuda(), torch.from_numpy(K).cuda()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    Sc = torch.einsum("ij,hid,hjd->hij", M, Qt, Kt)
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    H, m, n = 16, 8192, 8192
    assert isinstance(Sc, st.Tensor)
    assert Sc.format.levels == (st.LevelFormat.DENSE, st.LevelFormat.DENSE, st.LevelFormat.COMPRESSED)
    assert st.nnz(Sc) == H * Mh.nnz
    assert peak < H * m * n * 4 / 8, f"peak {peak / 2**30:.2f} GiB: a dense score tensor was materialised"
    vals = Sc.storage.values.reshape(H, -1)
    for h in (0, 9, 15):
        want = native.sddmm_csr(Mh.rowptr, Mh.colidx, Mh.vals, Q[h], K[h])
        bound = native.sddmm_csr(Mh.rowptr, Mh.colidx, Mh.vals, np.abs(Q[h]), np.abs(K[h]))
        rows = np.repeat(np.arange(m), np.diff(Mh.rowptr))
        lim = np.zeros(m)
        np.maximum.at(lim, rows, bound)
        assert np.all(np.abs(vals[h].cpu().numpy() - want) <= 1e-5 * lim[rows])


def test_repeated_calls_reuse_the_plan_and_rebind():
    r = np.random.default_rng(5)
    A = random_tensor(r, (60, 30), "csr", 0.2, "A")
    B1 = torch.randn(30, 8, device="cuda")
    B2 = torch.randn(30, 8, device="cuda")
    torch_dispatch._EXPRS.clear()
    y1 = torch.mm(A, B1)
    y2 = torch.mm(A, B2)
    assert len(torch_dispatch._EXPRS) == 1
    Ad = torch.from_numpy(st.to_dense(A)).cuda().float()
    torch.testing.assert_close(y1, Ad @ B1, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(y2, Ad @ B2, rtol=1e-5, atol=1e-5)
    # the cached expression holds no operand buffers
    (e,) = torch_dispatch._EXPRS.values()
    assert all(a.tensor.storage.values.numel() == 0 for a in e.accesses)


def test_out_keyword_and_rejected_arguments():
    r = np.random.default_rng(6)
    A = random_tensor(r, (20, 10), "csr", 0.3, "A")
    B = torch.randn(10, 4, device="cuda")
    out = torch.empty(20, 4, device="cuda")
    got = torch.mm(A, B, out=out)
    assert got is out
    torch.testing.assert_close(out, torch.from_numpy(st.to_dense(A)).cuda().float() @ B, rtol=1e-5, atol=1e-5)
    with pytest.raises(RuntimeError):
        torch.mm(A, B, out=torch.empty(3, 3, device="cuda"))
    with pytest.raises(TypeError):
        torch.add(A, 1.0)


def test_public_api_matches_oracle_on_cfg2_through_torch_mm():
    A, X, W1, _ = synthetic.cfg2()
    At = st.csr_from_arrays(A.rowptr, A.colidx, A.vals, A.shape, name="A")
    torch.backends.cuda.matmul.allow_tf32 = False
    Z = torch.from_numpy(X).cuda() @ torch.from_numpy(W1).cuda()
    got = torch.mm(At, Z).cpu().numpy()
    z = Z.double().cpu().numpy()
    rows = (0, 4096)  # the hub rows, where the merge carries are
    want = native.spmm_csr(A.rowptr, A.colidx, A.vals.astype(np.float64), z, rows=rows)
    bound = native.spmm_csr(A.rowptr, A.colidx, np.abs(A.vals.astype(np.float64)), np.abs(z), rows=rows)
    assert parity_gate(got[rows[0]:rows[1]], want, bound, 1e-5)[0]
