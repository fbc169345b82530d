"""Check the in-process group's collectives in isolation (diagnostics)."""
import ctypes as C
import sys
import threading
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
L = utv.lib()
f = L.utv_debug_collective
f.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
f.restype = C.c_int
hs = utv.local_group(P)
n = 1000
bufs = [torch.full((n,), float(p + 1), dtype=torch.float64, device="cuda") + torch.arange(n, device="cuda") for p in range(P)]
recvs = [torch.zeros(P * n, dtype=torch.float64, device="cuda") for _ in range(P)]
torch.cuda.synchronize()
ref_sum = sum(b.clone() for b in bufs)
ref_gather = torch.cat([b.clone() for b in bufs])
st = [None] * P


def run(op, root=0):
    def w(p):
        st[p] = f(hs[p].h, op, C.c_void_p(bufs[p].data_ptr()), n, root, C.c_void_p(recvs[p].data_ptr()))
    ts = [threading.Thread(target=w, args=(p,)) for p in range(P)]
    [t.start() for t in ts]
    [t.join(60) for t in ts]
    torch.cuda.synchronize()
    return st


print("allgather", run(2), [bool((r == ref_gather).all()) for r in recvs])
print("allreduce", run(0), [bool((b == ref_sum).all()) for b in bufs])
ref = bufs[1].clone() * 0 + 7.0
bufs[1].fill_(7.0); torch.cuda.synchronize()
print("bcast", run(1, root=1), [bool((b == 7.0).all()) for b in bufs])
