import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2405_16883_b200 as st
from paper_2405_16883_b200 import synthetic
A, X, W1, _ = synthetic.cfg2()
At = st.csr_from_arrays(A.rowptr, A.colidx, A.vals, A.shape, name="A")
Zt = st.from_dense(torch.from_numpy(X).cuda() @ torch.from_numpy(W1).cuda(), name="Z")
e = st.parse("H(i,k) = A(i,j) * Z(j,k)", {"A": At, "Z": Zt})
for _ in range(3): st.run(e)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): st.run(e)
torch.cuda.synchronize()
print("st.run cfg2 per call ms", (time.perf_counter() - t0) / 20 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): st.run(e)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
