import sys, ctypes, numpy as np, torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0); L = utv.lib()
R = torch.triu(torch.randn(256, 256, dtype=torch.float64, device="cuda")).t().contiguous().t()
h.svd_small(R); h.svd_small(R); torch.cuda.synchronize()
buf = (ctypes.c_longlong * 256)(); L.utv_debug_jac_trace(buf)
t = np.array(buf).reshape(32, 8)[:30]
print("per round cycles: load %.0f inner %.0f store %.0f barrier %.0f total %.0f" % (
    np.median(t[:, 1] - t[:, 0]), np.median(t[:, 2] - t[:, 1]), np.median(t[:, 3] - t[:, 2]),
    np.median(t[:, 4] - t[:, 3]), np.median(t[1:, 0] - t[:-1, 0])))
