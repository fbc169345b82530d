import sys, torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
m, w = int(sys.argv[1]), int(sys.argv[2])
P0 = utv.colmajor_empty(m, w); P0.normal_()
for _ in range(3):
    P = P0.clone(); h.hqr(P)
torch.cuda.synchronize()
