import sys, torch
sys.path.insert(0, '.')
from paper_2405_16883_b200 import ops, synthetic
W, XT = synthetic.cfg3()
R, C, V = (torch.from_numpy(W.rowptr).int().cuda(), torch.from_numpy(W.colidx).int().cuda(), torch.from_numpy(W.vals).cuda())
Xt = torch.from_numpy(XT).cuda(); out = torch.empty((W.shape[0], 4096), device='cuda')
for _ in range(2): ops.spmm_csr(R, C, V, Xt, out=out, variant='coltile')
torch.cuda.synchronize()
