"""One 256 x 256 Jacobi SVD (jacobi_kernel) for ncu."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
R = torch.triu(torch.randn(256, 256, dtype=torch.float64, device="cuda")).t().contiguous().t()
for _ in range(2):
    h.svd_small(R)
torch.cuda.synchronize()
