import sys, torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
R = torch.triu(torch.randn(256, 256, dtype=torch.float64, device="cuda")).t().contiguous().t()
for _ in range(2):
    Us, s, Vs, sw = h.svd_small(R)
torch.cuda.synchronize()
print("sweeps", sw)
