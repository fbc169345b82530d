"""The multi-GPU orchestration (paper_2408_05238_b200.dist) with the product backend on one GPU.

Only one GPU is available to this build's tests, so the NCCL path runs at world_size 1 (the
collectives are exercised through torch.distributed / NCCL with a single rank); the P > 1
schedule is covered on CPU over gloo (tests/test_dist_cpu.py) by the same orchestration code.
"""
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
import utv_inputs as gen

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p


@pytest.fixture(scope="module")
def utv():
    from paper_2408_05238_b200 import build
    build.build()
    import paper_2408_05238_b200 as m
    return m


@pytest.mark.parametrize("init_nccl", [False, True])
def test_dist_path_single_gpu(utv, init_nccl):
    from paper_2408_05238_b200 import dist as D
    if init_nccl:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda:0"))
    try:
        m, n, r, b, q = 700, 600, 290, 128, 2
        G = gen.GpMatrix(m, n, r, seed=21)
        B, X0 = G.known_rhs(k=2)
        A = torch.from_numpy(np.asfortranarray(G.A)).cuda()
        A_loc = D.scatter_columns(A, b, 1, 0)
        X, rk = D.lstsq_dist(A_loc, torch.from_numpy(B).cuda(), n, b=b, q=q, tau=1e-10, seed=5)
        Xo, ro = oracle.lstsq(G.A, B, b=b, q=q, tau=1e-10, seed=5)
        assert rk == ro == r
        Xg = X.cpu().numpy()
        assert np.linalg.norm(Xg - Xo) <= 1e-9 * np.linalg.norm(Xo)
        assert np.linalg.norm(Xg - X0) <= 1e-10 * np.linalg.norm(X0)
    finally:
        if init_nccl:
            dist.destroy_process_group()
