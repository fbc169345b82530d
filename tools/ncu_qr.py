"""One 50000 x 32 sub-panel QR (a single qr2_kernel launch) for ncu."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
P0 = utv.colmajor_empty(50000, 32); P0.normal_()
for _ in range(3):
    P = P0.clone(); h.hqr(P)
torch.cuda.synchronize()
