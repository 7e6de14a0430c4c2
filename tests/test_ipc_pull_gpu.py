"""The fused all-gather -> GEMM across PROCESSES: two ranks (gloo for the
handle exchange) on the box's one GPU, each owning a row slice of B in a
libmpfk allocation exported with CUDA IPC (dist.PeerBSlices).  Every rank
opens the other's slice through cudaIpcOpenMemHandle and its GEMM kernel
pulls B's panels from both slices while computing its row shard of C.  No
kernel waits on another rank's kernel: the slices are uploaded before a
barrier and only read afterwards.  This covers the cross-process plumbing
(handles, peer mappings, per-rank counters) that a one-rank run cannot."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, W, m, k, n, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2101_06584_b200 as P
    from paper_2101_06584_b200.dist import PeerBSlices, shard_rows
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        P.set_device(0)
        ld = P.pad_columns(n)
        slices = PeerBSlices(W, k, ld)
        c0, c1 = slices.cuts[rank], slices.cuts[rank + 1]
        slices.upload(P.fill_baseline(W, c1 - c0, n, 2, wide=True, row0=c0).data)
        dist.barrier()  # every slice resident before anyone pulls
        r0, r1 = shard_rows(m, world, rank, align=16)
        rows = r1 - r0
        A = P.fill_baseline(W, rows, k, 1, wide=True, row0=r0)
        dA = torch.from_numpy(A.data).cuda()
        dB = torch.zeros((W, k, ld), dtype=torch.float64, device="cuda")
        dC = torch.zeros((W, max(rows, 1), ld), dtype=torch.float64, device="cuda")
        launches = slices.step(W, dA, dB, dC, rows, n, k, panel_rows=64, chunk_rows=8, mode=mode)
        torch.cuda.synchronize()
        q.put((rank, r0, r1, dC[:, :rows].cpu().numpy(), dB.cpu().numpy(), launches))
        dist.barrier()  # nobody unmaps a slice another rank may still read
        slices.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["copy", "pull", "staged"])
@pytest.mark.parametrize("W,m,k,n", [(2, 96, 200, 70), (4, 50, 131, 33)])
def test_two_process_ipc_fused_allgather(gpu_lib, W, m, k, n, mode):
    import oracle as O
    P = gpu_lib
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, W, m, k, n, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    A = P.fill_baseline(W, m, k, 1, wide=True)
    B = P.fill_baseline(W, k, n, 2, wide=True)
    want = O.ref_gemm(A.data, B.data, k, n)
    for rank, r0, r1, C, Bfull, launches in got:
        per = 2 if mode == "staged" else 1  # staged: K panels [0, 64), [64, k)
        assert launches == (per if r1 > r0 else 0)
        assert np.array_equal(C.view(np.uint64), want[:, r0:r1].view(np.uint64))
        if r1 > r0:  # the pulled B is the whole matrix, bit for bit
            assert np.array_equal(Bfull.view(np.uint64), B.data.view(np.uint64))
