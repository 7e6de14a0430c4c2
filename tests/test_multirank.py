"""The N > 1 path on the CPU with the gloo backend, world_size 2 (the GPU box
has one GPU): the product's row partition (paper_2101_06584_b200.dist) plus
the B replication and the C all-gather, with the per-rank GEMM done by the
oracle through the driver's compute hook.  The assembled C must be
bit-identical to the single-rank GEMM, exactly as the reference's worker
partition is (linalg.hpp:399-433, acceptance.cpp:363-395)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_06584_b200.dist import gather_c, shard_rows, sharded_gemm_step


def test_shard_rows_partition():
    for m in (1, 63, 64, 65, 1000, 8192):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_rows(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 <= a1
            for r0, r1 in spans:
                assert r0 % 64 == 0 or r0 == r1 == m
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, W, m, k, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        ld = (n + 3) & ~3
        A = O.orc_fill_baseline(W, m, k, 1, wide=W > 2)
        r0, r1 = shard_rows(m, world, rank, align=8)
        rows = r1 - r0
        dA = torch.from_numpy(np.ascontiguousarray(A[:, r0:r1]))
        dB = torch.zeros((W, k, ld), dtype=torch.float64)
        if rank == 0:
            dB.copy_(torch.from_numpy(O.orc_fill_baseline(W, k, n, 2, wide=W > 2)))
        dC = torch.zeros((W, max(rows, 1), ld), dtype=torch.float64)

        def oracle_gemm(W_, dA_, dB_, dC_, rows_, n_, k_, ld_):
            Cs = O.orc_gemm(dA_.numpy(), dB_.numpy(), k_, n_)
            dC_[:, :rows_] = torch.from_numpy(Cs)
            return 1

        launches = sharded_gemm_step(W, dA, dB, dC, rows, n, k, ld, gemm=oracle_gemm)
        Cfull = gather_c(dC[:, :rows], m, world, align=8)
        if rank == 0:
            want = O.orc_gemm(A, O.orc_fill_baseline(W, k, n, 2, wide=W > 2), k, n)
            same = np.array_equal(Cfull.numpy().view(np.uint64), want.view(np.uint64))
            q.put((same, launches))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W,m,k,n", [(2, 37, 21, 19), (3, 16, 9, 10), (4, 20, 7, 6)])
def test_two_rank_gloo_row_shards_bit_identical(W, m, k, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, W, m, k, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    same, launches = q.get(timeout=10)
    assert same and launches == 1


def _worker_overlapped(rank, world, port, W, m, k, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes as C

        import oracle as O
        from paper_2101_06584_b200.dist import sharded_gemm_step_overlapped
        ld = (n + 3) & ~3
        A = O.orc_fill_baseline(W, m, k, 1, wide=True)
        r0, r1 = shard_rows(m, world, rank, align=8)
        rows = r1 - r0
        dA = torch.from_numpy(np.ascontiguousarray(A[:, r0:r1]))
        dB = torch.zeros((W, k, ld), dtype=torch.float64)
        if rank == 0:
            dB.copy_(torch.from_numpy(O.orc_fill_baseline(W, k, n, 2, wide=True)))
        dC = torch.zeros((W, max(rows, 1), ld), dtype=torch.float64)

        def oracle_panel(W_, Ap, Bp, dC_, rows_, n_, kp, ld_, acc):
            a = np.ascontiguousarray(Ap.numpy())
            b = np.ascontiguousarray(Bp.numpy())
            if not acc:
                dC_[:, :rows_] = torch.from_numpy(O.orc_gemm(a, b, kp, n_))
            else:
                c = np.ascontiguousarray(dC_[:, :rows_].numpy())
                O.orc().orc_gemm_acc(W_, rows_, kp, n_, a.ctypes.data, a.shape[2], a.shape[1] * a.shape[2],
                                     b.ctypes.data, b.shape[2], b.shape[1] * b.shape[2], c.ctypes.data,
                                     c.shape[2], c.shape[1] * c.shape[2])
                dC_[:, :rows_] = torch.from_numpy(c)
            return 1

        launches = sharded_gemm_step_overlapped(W, dA, dB, dC, rows, n, k, ld, panels=3, gemm=oracle_panel)
        Cfull = gather_c(dC[:, :rows], m, world, align=8)
        if rank == 0:
            want = O.orc_gemm(A, O.orc_fill_baseline(W, k, n, 2, wide=True), k, n)
            q.put((np.array_equal(Cfull.numpy().view(np.uint64), want.view(np.uint64)), launches))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W,m,k,n", [(2, 21, 50, 13), (4, 12, 40, 7)])
def test_two_rank_gloo_overlapped_k_panels(W, m, k, n):
    """B broadcast in K panels overlapped with per-panel continuation GEMMs:
    bit-identical to the one-shot product (linalg.hpp:261)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_overlapped, args=(r, 2, port, W, m, k, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    same, launches = q.get(timeout=10)
    from paper_2101_06584_b200.dist import k_panels
    assert same and launches == len(k_panels(k, 3)) > 1


def _oracle_panel(W_, Ap, Bp, dC_, rows_, n_, kp, ld_, acc):
    import oracle as O
    a = np.ascontiguousarray(Ap.numpy())
    b = np.ascontiguousarray(Bp.numpy())
    c = np.ascontiguousarray(dC_[:, :rows_].numpy())
    if not acc:
        c[...] = O.orc_gemm(a, b, kp, n_)[:, :, : c.shape[2]]
    else:
        O.orc().orc_gemm_acc(W_, rows_, kp, n_, a.ctypes.data, a.shape[2], a.shape[1] * a.shape[2],
                             b.ctypes.data, b.shape[2], b.shape[1] * b.shape[2], c.ctypes.data,
                             c.shape[2], c.shape[1] * c.shape[2])
    dC_[:, :rows_] = torch.from_numpy(c)
    return 1


def _worker_host(rank, world, port, W, m, k, n, panels, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_2101_06584_b200 import MPMatrix
        from paper_2101_06584_b200.dist import matmul_sharded_into
        Af = O.orc_fill_baseline(W, m, k, 1, wide=True)
        Bf = O.orc_fill_baseline(W, k, n, 2, wide=True)
        r0, r1 = shard_rows(m, world, rank, align=8)
        A = MPMatrix.from_planes(Af[:, r0:r1, :k])
        B = MPMatrix.from_planes(Bf[:, :, :n])
        Cs = MPMatrix(W, r1 - r0, n)
        Cs.data[...] = 7.0  # must be overwritten, pads included
        launches = matmul_sharded_into(Cs, A, B, panels=panels, device=torch.device("cpu"), gemm=_oracle_panel)
        Cfull = gather_c(torch.from_numpy(Cs.data), m, world, align=8)
        if rank == 0:
            want = O.orc_gemm(Af, Bf, k, n)
            q.put((np.array_equal(Cfull.numpy().view(np.uint64), want.view(np.uint64)), launches))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,W,m,k,n,panels", [(2, 2, 21, 50, 13, 3), (2, 3, 9, 70, 5, 2), (2, 4, 12, 33, 7, 8),
                                                  (2, 2, 5, 31, 6, 1), (3, 2, 30, 61, 9, 2), (3, 4, 7, 40, 5, 3)])
def test_gloo_host_operands_sliced_b(world, W, m, k, n, panels):
    """B starts on the host: each rank uploads 1/world of every K panel, the
    panels are all-gathered, the shard GEMM continues panel by panel; the
    assembled C is bit-identical to the one-shot product, including ragged
    last panels (k not a multiple of the panel height) and ranks without
    rows."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_host, args=(r, world, port, W, m, k, n, panels, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs)
    same, launches = q.get(timeout=10)
    from paper_2101_06584_b200.dist import gather_panels
    assert same and launches == len(gather_panels(k, panels, world)[1])


def test_gather_panels_plan():
    from paper_2101_06584_b200.dist import gather_panels
    for k in (1, 15, 16, 100, 8192, 8193):
        for world in (1, 2, 8):
            for panels in (1, 3, 8):
                pk, parts = gather_panels(k, panels, world)
                assert pk % (16 * world) == 0
                assert parts[0][0] == 0 and parts[-1][1] == k
                assert all(b - a <= pk and a % pk == 0 for a, b in parts)
                assert len(parts) <= panels or pk == 16 * world
    assert gather_panels(0, 4, 2)[1] == []
