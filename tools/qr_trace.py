import sys, ctypes, numpy as np, torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
L = utv.lib()
for m in (50000, 2000):
    P0 = utv.colmajor_empty(m, 32); P0.normal_()
    for _ in range(2):
        P = P0.clone(); h.hqr(P)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 1024)()
    L.utv_debug_qr_trace(buf)
    t = np.array(buf[:512]).reshape(64, 8)[:32]
    # phases: 0 loop start, 3 after block reduce, 4 after barrier, 1 after partial reduce, 2 after dlarfg/T
    d = lambda a, b: t[:, b] - t[:, a]
    print(m, "cycles/col: reduce_store %.0f barrier %.0f partials %.0f dlarfg+T %.0f update %.0f total %.0f" % (
        np.median(d(0, 3)), np.median(d(3, 4)), np.median(d(4, 1)), np.median(d(1, 2)),
        np.median(t[1:, 0] - t[:-1, 2]), np.median(t[1:, 0] - t[:-1, 0])))
