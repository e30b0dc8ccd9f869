"""Public-call overhead of the drop-in API on cfg2 (st.run / torch.mm vs the kernel alone).

python tools/api_overhead_probe.py [--profile]  -> per-call host time of N back-to-back calls
(no synchronisation inside the loop) against the device time of the SpMM kernel itself."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2405_16883_b200 as st  # noqa: E402
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402

A, X, W1, _ = synthetic.cfg2()
At = st.csr_from_arrays(A.rowptr, A.colidx, A.vals, A.shape, name="A")
Zd = torch.from_numpy(X).cuda() @ torch.from_numpy(W1).cuda()
Zt = st.from_dense(Zd, name="Z")
e = st.parse("H(i,k) = A(i,j) * Z(j,k)", {"A": At, "Z": Zt})
N = 200


def per_call_us(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / N * 1e6


def kernel_us():
    L = At.storage.levels[1]
    out = torch.empty_like(Zd)
    st.run(e)  # builds the cached plan
    part = At._cache[("partition", 128, 0)]
    stats = At._cache[("stats", 0)]
    fn = lambda: ops.spmm_csr(L.pos, L.crd, At.storage.values, Zd, out=out, variant="merge",  # noqa: E731
                              partition=part, stats=stats)
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    s.record()
    for _ in range(N):
        fn()
    t.record()
    torch.cuda.synchronize()
    return s.elapsed_time(t) / N * 1e3, per_call_us(fn)


k_dev, k_host = kernel_us()
r = per_call_us(lambda: st.run(e))
mm = per_call_us(lambda: torch.mm(At, Zd))
mat = per_call_us(lambda: At @ Zd)
print(f"cfg2 SpMM: kernel {k_dev:.1f} us device/call back to back; ops.spmm_csr {k_host:.1f} us/call; "
      f"st.run {r:.1f} us/call; torch.mm(A, Z) {mm:.1f} us/call; A @ Z {mat:.1f} us/call")
print(f"overhead over the kernel: st.run {r - k_dev:+.1f} us, torch.mm {mm - k_dev:+.1f} us")
if "--profile" in sys.argv:
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        st.run(e)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)

# small operand (cfg1, 4096^2 at 1 %, K = 64): host cost per call is no longer hidden by the kernel
A1, B1 = synthetic.cfg1()
A1t = st.csr_from_arrays(A1.rowptr, A1.colidx, A1.vals, A1.shape, name="A")
B1d = torch.from_numpy(B1).cuda()
e1 = st.parse("C(i,k) = A(i,j) * B(j,k)", {"A": A1t, "B": st.from_dense(B1d, name="B")})
st.run(e1)
L1 = A1t.storage.levels[1]
s_, t_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s_.record()
for _ in range(N):
    ops.spmm_csr(L1.pos, L1.crd, A1t.storage.values, B1d, variant="row")
t_.record()
torch.cuda.synchronize()
k1 = s_.elapsed_time(t_) / N * 1e3
print(f"cfg1 SpMM: kernel {k1:.1f} us device/call; ops.spmm_csr {per_call_us(lambda: ops.spmm_csr(L1.pos, L1.crd, A1t.storage.values, B1d, variant='row')):.1f} us/call; "
      f"st.run {per_call_us(lambda: st.run(e1)):.1f} us/call; torch.mm {per_call_us(lambda: torch.mm(A1t, B1d)):.1f} us/call")
