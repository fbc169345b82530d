import sys, ctypes, numpy as np, torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0); L = utv.lib()
P0 = utv.colmajor_empty(50000, 32); P0.normal_()
for _ in range(3):
    P = P0.clone(); h.hqr(P)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 1024)()
L.utv_debug_qr_trace(buf)
a = np.array(buf[512:512 + 132]); d = np.array(buf[768:768 + 132])
a0 = a.min()
print("arrival spread ns: min 0, median %d, max %d; argmax CTA %d" % (np.median(a - a0), (a - a0).max(), (a - a0).argmax()))
print("departure: first %d, median %d, last %d" % ((d - a0).min(), np.median(d - a0), (d - a0).max()))
print("arrivals by CTA (ns):", list((a - a0)[:: 11]))
