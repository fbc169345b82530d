"""The panel QR's inter-sub-panel GEMM shapes (50000 rows) under every tile config x split-K:
TN  P_r^T W_b  (M = wr, N = 32, K = m')   and   NT  P_r -= W_b Z2^T  (M = m', N = wr, K = 32)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv  # noqa: E402

h = utv.Handle(0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 50000


def timeit(f, reps=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h.stream)
        f()
        e1.record(h.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]


res = []
for wr in (224, 96):
    P = utv.colmajor_empty(m, wr).normal_()
    W = utv.colmajor_empty(m, 32).normal_()
    Z = utv.colmajor_empty(wr, 32).normal_()
    Ct = utv.colmajor_empty(wr, 32)
    for kind in ("TN", "NT"):
        best = None
        for cfg in (-1, 0, 1, 2, 3, 4, 5):
            for sp in ((0, 1, 2, 4, 8, 16, 32, 64, 128, 256) if kind == "TN" else (0, 1)):
                with utv.tuned(utv.UTV_TUNE_GEMM_CFG, cfg, utv.UTV_TUNE_GEMM_SPLITS, sp):
                    if kind == "TN":
                        f = lambda: h.gemm(True, False, 1.0, P, W, 0.0, Ct)          # noqa: E731
                    else:
                        f = lambda: h.gemm(False, True, -1.0, W, Z, 1.0, P)          # noqa: E731
                    try:
                        t = timeit(f)
                    except Exception as e:          # noqa: BLE001
                        continue
                res.append({"kind": kind, "wr": wr, "cfg": cfg, "splits": sp, "us": t})
                if best is None or t < best[0]:
                    best = (t, cfg, sp)
                if cfg == -1 and sp == 0:
                    auto = t
        print(f"{kind} wr={wr}: automatic {auto:.1f} us, best {best[0]:.1f} us at cfg {best[1]} splits {best[2]}", flush=True)
json.dump(res, open("gpurun_out/skinny_gemm_sweep.json", "w"), indent=1)
