"""In-situ execution time of the side-stream Jacobi SVD kernel during one cfg lstsq call
(CTA 0's %globaltimer at kernel entry / exit, utv_debug_jac_times), against the stream-event
window of the SVD family (which also counts the wait for a free 8-SM cluster slot).
usage: python tools/jac_insitu.py [cfg3|cfg2]"""
import ctypes, json, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paper_2408_05238_b200 as utv
import utv_inputs as gen

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
m, n, r_true, b, q, k = bench.CONFIGS[cfg]
dev = torch.device("cuda:0")
opts = utv.Opts(block=b, power_iters=q, tau=1e-10, seed=gen.SKETCH_SEED)
At, Bm, X0 = gen.gp_torch(m, n, r_true, seed=gen.MATRIX_SEED, device=dev, k=k)
A0 = At.t(); B0 = utv.colmajor(Bm)
h = utv.Handle(0)
A = utv.colmajor_empty(m, n); B = utv.colmajor_empty(m, k); X = utv.colmajor_empty(n, k)
lib = utv.lib()
lib.utv_debug_jac_times.restype = ctypes.c_int
lib.utv_debug_jac_times.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = np.zeros(2 * 4096, dtype=np.uint64)
def step():
    A.copy_(A0); B.copy_(B0); return h.lstsq(A, B, X, opts)
step(); torch.cuda.synchronize()
lib.utv_debug_jac_times(buf.ctypes.data, 0, 1)
h.profile(True)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(h.stream); step(); e1.record(h.stream); torch.cuda.synchronize()
total_ms = e0.elapsed_time(e1)
cnt = lib.utv_debug_jac_times(buf.ctypes.data, 4096, 1)
d = (buf[1:2 * cnt:2].astype(np.int64) - buf[0:2 * cnt:2].astype(np.int64)) / 1e6
prof = h.profile_read()
svd_ev = prof["svd"]["ms"]
res = {"config": cfg, "step_ms": total_ms, "jacobi_launches": cnt, "jacobi_exec_ms_total": float(d.sum()),
       "jacobi_exec_ms_first": float(d[0]), "jacobi_exec_ms_median": float(np.median(d)),
       "jacobi_exec_ms_max": float(d.max()), "svd_family_event_ms": svd_ev,
       "exec_first10": [round(float(x), 2) for x in d[:10]], "exec_last10": [round(float(x), 2) for x in d[-10:]],
       "sm_ms_share": float(d.sum()) * 8 / 148 / total_ms}
print(json.dumps(res, indent=1))
json.dump(res, open(f"gpurun_out/jac_insitu_{cfg}.json", "w"), indent=1)
