"""Per-step cost of the e2e path's compute part alone (inputs already on the device): wrapping the
uploaded graph as a declared CSR tensor and the GCN forward through torch.mm interception (plan +
SpMM) -- the part of bench.py's e2e step that overlaps the PCIe copies."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2405_16883_b200 as st  # noqa: E402
from paper_2405_16883_b200 import synthetic  # noqa: E402

A, X, W1, W2 = synthetic.cfg2()
dev = torch.device("cuda")
rp, ci, v = (torch.from_numpy(a).to(dev) for a in (A.rowptr.astype(np.int32), A.colidx.astype(np.int32), A.vals))
x, w1, w2 = (torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev) for a in (X, W1, W2))


def step(fresh=True):
    At = st.csr_from_arrays(rp, ci, v, A.shape, name="A", device=dev, validate=False)
    H = torch.relu_(torch.mm(At, x @ w1))
    return torch.mm(At, H @ w2)


for label in ("fresh tensor per step (bench e2e)",):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    n = 20
    for _ in range(n):
        step()
    e.record()
    torch.cuda.synchronize()
    print(f"{label}: {s.elapsed_time(e) / n:.3f} ms/step device, {(time.perf_counter() - t0) / n * 1e3:.3f} ms/step wall")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
