"""Multi-GPU orchestration checked on CPU: world_size 2 and 3 over gloo.

The block-cyclic layout, the AllReduce / AllGather / Broadcast schedule and the distributed
block back substitution of paper_2408_05238_b200.dist run with the CPU step backend
(tests/dist_cpu_backend.py); the gathered x must match the single-process oracle to 1e-9 with an
identical rank.  The same orchestration runs on GPUs with dist.CudaSteps over NCCL.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    import utv_inputs as gen
    from paper_2408_05238_b200 import dist as D
    from dist_cpu_backend import CpuSteps
    torch.set_num_threads(1)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    m, n, r, b, q, k = case
    G = gen.GpMatrix(m, n, r, seed=m + n)
    B, _ = G.known_rhs(k=k, consistent=m < 2 * r)
    A = torch.from_numpy(np.asfortranarray(G.A))
    A_loc = D.scatter_columns(A, b, world, rank)
    X, rk = D.lstsq_dist(A_loc, torch.from_numpy(B), n, b=b, q=q, tau=1e-10, seed=7, steps=CpuSteps())
    np.save(os.path.join(outdir, f"x{rank}.npy"), X.numpy())
    np.save(os.path.join(outdir, f"r{rank}.npy"), np.array([rk]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [(260, 200, 90, 32, 1, 2), (300, 300, 150, 64, 2, 1), (150, 110, 110, 16, 1, 1)])
def test_dist_matches_oracle(tmp_path, world, case):
    import oracle
    import utv_inputs as gen
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    m, n, r, b, q, k = case
    G = gen.GpMatrix(m, n, r, seed=m + n)
    B, _ = G.known_rhs(k=k, consistent=m < 2 * r)
    Xo, ro = oracle.lstsq(G.A, B, b=b, q=q, tau=1e-10, seed=7)
    for rank in range(world):
        X = np.load(tmp_path / f"x{rank}.npy")
        rk = int(np.load(tmp_path / f"r{rank}.npy")[0])
        assert rk == ro
        assert np.linalg.norm(X - Xo) <= 1e-9 * np.linalg.norm(Xo)


def test_scatter_gather_roundtrip():
    from paper_2408_05238_b200 import dist as D
    A = torch.arange(7 * 23, dtype=torch.float64).reshape(23, 7).t().contiguous().t()   # 7 x 23 col-major
    A = torch.randn(9, 23, dtype=torch.float64)
    for P in (1, 2, 3, 4):
        shards = [D.scatter_columns(A, 4, P, p) for p in range(P)]
        assert sum(s.shape[1] for s in shards) == 23
        assert torch.equal(D.gather_columns(shards, 23, 4), A)
