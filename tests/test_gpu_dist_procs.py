"""The NATIVE multi-GPU path (lstsq_dist / lstsq_dist_ooc in libutv.so) across separate PROCESSES.

One process per rank -- the deployment shape of the multi-GPU path -- with the collectives
supplied by the caller through utv_create_with_comm (here torch.distributed over gloo, staged
through host memory by the binding); every process runs its rank on cuda:0, the one GPU of this
pool.  This is the same C++ orchestration that runs over NCCL with utv_create_dist (only the
transport differs), so the block-cyclic layout, the collective sequence and the owner logic are
exercised with separate address spaces.  Gates: r identical on every rank and equal to the
oracle's, X bit-identical on every rank and within 1e-9 of the oracle.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, streamed, outdir):
    sys.path.insert(0, ROOT)
    import utv_inputs as gen
    import paper_2408_05238_b200 as utv
    from paper_2408_05238_b200 import dist as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    m, n, r, b, q, k = case
    G = gen.GpMatrix(m, n, r, seed=m + n + world)
    B, _ = G.known_rhs(k=k)
    B = B.reshape(m, -1)
    Ad = torch.from_numpy(np.ascontiguousarray(G.A.T)).cuda().t()
    sh = D.scatter_columns(Ad, b, world, rank)
    nloc = sh.shape[1]
    if streamed:
        A = utv.colmajor_empty(m, max(nloc, 1), device="cpu", pin_memory=True)
        A[:, :nloc].copy_(sh)
    else:
        A = utv.colmajor_empty(m, max(nloc, 1))
        A[:, :nloc].copy_(sh)
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().t()
    X = utv.colmajor_empty(n, B.shape[1])
    h = utv.comm_handle(rank, world)
    flags = utv.UTV_HOST_STREAMED if streamed else 0
    rk = h.lstsq(A, Bd, X, utv.Opts(block=b, power_iters=q, tau=1e-10, seed=3, flags=flags))
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, f"x{rank}.npy"), X.cpu().numpy())
    np.save(os.path.join(outdir, f"r{rank}.npy"), np.array([rk]))
    h.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case,streamed", [
    (2, (600, 600, 300, 64, 1, 2), False),
    (3, (700, 550, 260, 64, 2, 1), False),      # ragged last block
    (2, (2048, 2048, 1000, 256, 2, 1), False),  # b = 256: the cluster Jacobi and the fused update
    (2, (640, 512, 200, 64, 1, 1), True),       # out-of-core shards (UTV_HOST_STREAMED)
])
def test_native_multiprocess_matches_oracle(tmp_path, monkeypatch, world, case, streamed):
    import oracle
    import utv_inputs as gen
    if streamed:
        monkeypatch.setenv("UTV_OOC_MAX_RESIDENT_COLS", "0")
    mp.spawn(_worker, args=(world, _free_port(), case, streamed, str(tmp_path)), nprocs=world, join=True)
    m, n, r, b, q, k = case
    G = gen.GpMatrix(m, n, r, seed=m + n + world)
    B, X0 = G.known_rhs(k=k)
    Xo, ro = oracle.lstsq(G.A, B.reshape(m, -1), b=b, q=q, tau=1e-10, seed=3)
    Xs = [np.load(tmp_path / f"x{p}.npy") for p in range(world)]
    rs = [int(np.load(tmp_path / f"r{p}.npy")[0]) for p in range(world)]
    assert rs == [ro] * world and ro == r, (rs, ro)
    for X in Xs:
        assert np.array_equal(X, Xs[0])                              # replicated result, bit-identical
    assert np.linalg.norm(Xs[0] - Xo) <= 1e-9 * np.linalg.norm(Xo)
    assert np.linalg.norm(Xs[0] - X0.reshape(Xs[0].shape)) <= 1e-10 * np.linalg.norm(X0)
