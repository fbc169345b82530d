"""Host vs device time of launch-heavy calls (is the host the bottleneck for small-kernel chains?)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
for m, w in ((256, 256), (2000, 256), (20000, 256)):
    P0 = utv.colmajor_empty(m, w); P0.normal_()
    Ps = [P0.clone() for _ in range(20)]
    h.hqr(Ps[0]); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for P in Ps:
        h.hqr(P)
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"hqr {m}x{w}: host enqueue {(t1 - t0) / 20 * 1e3:.3f} ms/call, device {e0.elapsed_time(e1) / 20:.3f} ms/call, wall {(t2 - t0) / 20 * 1e3:.3f}", flush=True)
A = utv.colmajor_empty(64, 64); A.normal_(); B = utv.colmajor_empty(64, 64); B.normal_(); Cm = utv.colmajor_empty(64, 64)
h.gemm(False, False, 1.0, A, B, 0.0, Cm); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    h.gemm(False, False, 1.0, A, B, 0.0, Cm)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"tiny gemm: host {(t1 - t0) / 2000 * 1e6:.1f} us/call (incl. Python/ctypes), wall {(t2 - t0) / 2000 * 1e6:.1f} us/call")
