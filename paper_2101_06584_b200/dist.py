"""Multi-GPU row-sharded GEMM: one process per GPU over torch.distributed.

The reference parallelises matmul_block_parallel_into over threads that own
disjoint contiguous spans of row blocks and never exchange data
(linalg.hpp:399-433).  Here each rank (GPU) owns a contiguous span of rows of
A and C; the only exchange is the replication of B from the root rank to every
GPU (NCCL broadcast over NVLink/NVSwitch), then each rank runs the sm_100a
GEMM on its shard.  No reduction follows: rows of C are independent and every
element's accumulation order is the reference's, so the result is
bit-identical for any world size.  An optional all-gather assembles a
replicated C when a caller needs one.
"""
from __future__ import annotations

from typing import Callable, Optional


def shard_rows(m: int, world: int, rank: int, align: int = 64):
    """Contiguous row span [r0, r1) of `rank`: ceil-divided blocks of `align`
    rows, like the reference's `per = ceil(nblocks / nt)` spans
    (linalg.hpp:413-421).  Trailing ranks may get an empty span."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_rows: bad rank/world")
    nblocks = (m + align - 1) // align
    per = (nblocks + world - 1) // world
    r0 = min(m, rank * per * align)
    r1 = min(m, (rank + 1) * per * align)
    return r0, r1


def replicate_b(dB, src: int = 0, group=None):
    """B from the root rank to all ranks (NCCL broadcast on GPU tensors)."""
    import torch.distributed as dist
    if dist.is_initialized():
        dist.broadcast(dB, src=src, group=group)
    return dB


def sharded_gemm_step(W: int, dA, dB, dC, rows: int, n: int, k: int, ld: int, *, stream=None,
                      gemm: Optional[Callable] = None, group=None) -> int:
    """One step of the sharded GEMM on this rank: replicate B, then
    C_shard = A_shard * B.  dA (W, rows, ld), dB (W, k, ld), dC (W, rows, ld)
    float64 tensors.  `gemm` defaults to libmpfk's device entry point;
    returns the number of GEMM kernel launches."""
    replicate_b(dB, group=group)
    if rows == 0:
        return 0
    if gemm is None:
        from . import linalg as L
        s = stream.cuda_stream if stream is not None else 0
        lda, ldb, ldc = dA.shape[2], dB.shape[2], dC.shape[2]
        return L.gemm_device(W, rows, n, k, dA.data_ptr(), lda, dA.shape[1] * lda, dB.data_ptr(), ldb,
                             dB.shape[1] * ldb, dC.data_ptr(), ldc, dC.shape[1] * ldc, s)
    return gemm(W, dA, dB, dC, rows, n, k, ld)


def k_panels(k: int, panels: int, align: int = 16):
    """Split [0, k) into <= panels contiguous K panels whose starts are
    multiples of `align` (even offsets keep 16-byte cp.async rows)."""
    panels = max(1, min(panels, k // align if k >= align else 1))
    pk = ((k + panels - 1) // panels + align - 1) // align * align
    return [(k0, min(k, k0 + pk)) for k0 in range(0, k, pk)] or [(0, 0)]


def sharded_gemm_step_overlapped(W: int, dA, dB, dC, rows: int, n: int, k: int, ld: int, *, panels: int = 4,
                                 stream=None, gemm: Optional[Callable] = None, group=None) -> int:
    """One sharded step with the B replication overlapped with compute: B is
    broadcast in K panels (one asynchronous NCCL broadcast per panel and
    component plane, all queued at once), and the rank's GEMM runs panel by
    panel -- panel 0 with mpfk_gemm_device, later panels with
    mpfk_gemm_device_acc continuing the chains stored in C -- each launch
    gated only on its own panel's broadcast.  Bit-identical to
    sharded_gemm_step (the chain state between k steps is exactly C,
    linalg.hpp:261).

    `gemm(W, A_panel, B_panel, dC, rows, n, kp, ld, accumulate)` overrides
    the device kernel (the CPU tests pass the oracle)."""
    import torch.distributed as dist
    parts = k_panels(k, panels)
    multi = dist.is_initialized()  # (a world of one still runs the collective path)
    works = []
    if multi:
        for k0, k1 in parts:
            works.append([dist.broadcast(dB[w, k0:k1], src=0, group=group, async_op=True) for w in range(W)])
    launches = 0
    for p, (k0, k1) in enumerate(parts):
        if multi:
            for wk in works[p]:
                wk.wait()  # the compute stream waits for this panel only
        if rows == 0 or k1 == k0:
            continue
        if gemm is not None:
            launches += gemm(W, dA[:, :, k0:k1], dB[:, k0:k1], dC, rows, n, k1 - k0, ld, p > 0)
            continue
        from . import linalg as L
        s = stream.cuda_stream if stream is not None else 0
        f = L.gemm_device if p == 0 else L.gemm_device_acc
        lda, ldb, ldc = dA.shape[2], dB.shape[2], dC.shape[2]
        launches += f(W, rows, n, k1 - k0, dA.data_ptr() + 8 * k0, lda, dA.shape[1] * lda,
                      dB.data_ptr() + 8 * k0 * ldb, ldb, dB.shape[1] * ldb, dC.data_ptr(), ldc,
                      dC.shape[1] * ldc, s)
    return launches


def gather_panels(k: int, panels: int, world: int, align: int = 16):
    """K panel plan for B starting on the host: panel height pk is a multiple
    of align*world so every panel splits into `world` equal sub-slices of
    pk/world rows, rank r uploading sub-slice r.  Returns (pk, [(k0, k1)]);
    the last panel may be short (k1 - k0 < pk), its missing rows zero."""
    if k <= 0:
        return align * world, []
    panels = max(1, panels)
    unit = align * world
    pk = max(unit, ((k + panels - 1) // panels + unit - 1) // unit * unit)
    return pk, [(k0, min(k, k0 + pk)) for k0 in range(0, k, pk)]


def matmul_sharded_into(C_, A, B, *, panels: int = 8, group=None, device=None,
                        gemm: Optional[Callable] = None) -> int:
    """This rank's row shard of C = A*B with every operand starting and
    ending in host memory: the multi-process counterpart of
    matmul_block_parallel_into (linalg.hpp:402-433), one rank per GPU.

    A, C_: this rank's row shard (host MPMatrix, pinned for overlap); B: the
    whole K x n right operand, readable by every rank (e.g. an MPFM file
    mapped on each).  Each rank copies only 1/world of B over its own PCIe
    link -- sub-slice r of each K panel ("each GPU H2D-copies
    B's 1/G slice, then all-gather") -- and the panels are assembled on every
    GPU with NCCL all-gathers queued ahead of the compute.  The GEMM runs
    panel by panel (mpfk_gemm_device, then mpfk_gemm_device_acc continuing
    the chains kept in C, linalg.hpp:261), each launch waiting only for its
    own panel, so the host copies and NVLink traffic overlap the FP64 work.
    The shard of C is bit-identical to the single-GPU product for any world
    size.  Collective: every rank of `group` must call it (a rank with no
    rows passes 0-row A and C).  Returns the number of GEMM launches.

    `gemm(W, A_panel, B_panel, dC, rows, n, kp, ld, accumulate)` overrides
    the device kernel (the CPU tests pass the oracle)."""
    import torch
    import torch.distributed as dist
    from . import linalg as L
    L._check_same_width(C_, A, B)
    if A.cols() != B.rows():
        raise ValueError("matmul: inner dimensions differ")
    if C_.rows() != A.rows() or C_.cols() != B.cols():
        raise ValueError("matmul: result shape mismatch")
    W, rows, k, n = A.W, A.rows(), A.cols(), B.cols()
    multi = dist.is_initialized()
    world = dist.get_world_size(group) if multi else 1
    rank = dist.get_rank(group) if multi else 0
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else \
            torch.device("cpu")
    cuda = device.type == "cuda"
    if gemm is None and not cuda:
        raise RuntimeError("matmul_sharded_into: the GEMM runs on a CUDA device (there is no CPU path)")
    ld = B.stride()
    pk, parts = gather_panels(k, panels, world)
    chunk = pk // world
    f64 = torch.float64
    dB = torch.empty((W, max(1, len(parts)) * pk, ld), dtype=f64, device=device)
    piece = torch.zeros((max(1, len(parts)), W, chunk, ld), dtype=f64, device=device)
    ldc = C_.stride()
    dC = torch.zeros((W, max(rows, 1), ldc), dtype=f64, device=device)
    dA = torch.empty((W, max(rows, 1), A.stride()), dtype=f64, device=device)
    hA, hB, hC = torch.from_numpy(A.data), torch.from_numpy(B.data), torch.from_numpy(C_.data)
    comp = torch.cuda.current_stream(device) if cuda else None
    up = torch.cuda.Stream(device) if cuda else None
    down = torch.cuda.Stream(device) if cuda else None

    def mark(stream):
        if not cuda:
            return None
        e = torch.cuda.Event()
        e.record(stream)
        return e

    # host -> device on the copy stream, in the order the GEMMs consume it:
    # A's shard, then this rank's sub-slice of each K panel (one contiguous
    # copy per plane), each panel all-gathered as soon as its slice is in
    works, ready = [], []
    with (torch.cuda.stream(up) if cuda else _null_ctx()):
        if cuda:
            up.wait_stream(comp)  # the zero fills above
        if rows:
            dA[:, :rows].copy_(hA, non_blocking=cuda)
        a_ready = mark(up)
        for p, (k0, _k1) in enumerate(parts):
            s0 = k0 + rank * chunk
            s1 = min(k, s0 + chunk)
            for w in range(W):
                if s1 > s0:
                    piece[p, w, : s1 - s0].copy_(hB[w, s0:s1], non_blocking=cuda)
            if multi:
                works.append([dist.all_gather_into_tensor(dB[w, k0:k0 + pk], piece[p, w], group=group,
                                                          async_op=True) for w in range(W)])
            else:
                dB[:, k0:k0 + pk].copy_(piece[p])
                works.append([])
            ready.append(mark(up))
    if a_ready is not None:
        comp.wait_event(a_ready)

    # the last panel runs in row chunks so the download of C overlaps it
    tail = [(0, rows)]
    if cuda and rows >= 128:
        step = max(64, (rows // 4 + 63) // 64 * 64)
        tail = [(r, min(rows, r + step)) for r in range(0, rows, step)]
    launches = 0
    lda = dA.shape[2]
    for p, (k0, k1) in enumerate(parts):
        for wk in works[p]:
            wk.wait()  # the compute stream waits for this panel only
        if ready[p] is not None:
            comp.wait_event(ready[p])
        if rows == 0:
            continue
        if gemm is not None:
            launches += gemm(W, dA[:, :rows, k0:k1], dB[:, k0:k1], dC, rows, n, k1 - k0, ldc, p > 0)
            continue
        f = L.gemm_device if p == 0 else L.gemm_device_acc
        for r0, r1 in (tail if p == len(parts) - 1 else [(0, rows)]):
            launches += f(W, r1 - r0, n, k1 - k0, dA.data_ptr() + 8 * (r0 * lda + k0), lda, dA.shape[1] * lda,
                          dB.data_ptr() + 8 * k0 * ld, ld, dB.shape[1] * ld, dC.data_ptr() + 8 * r0 * ldc, ldc,
                          dC.shape[1] * ldc, comp.cuda_stream)
            if p == len(parts) - 1:
                done = mark(comp)
                down.wait_event(done)
                with torch.cuda.stream(down):
                    for w in range(W):
                        hC[w, r0:r1].copy_(dC[w, r0:r1], non_blocking=True)
    if rows and (gemm is not None or not parts):
        if cuda:
            down.wait_stream(comp)
        with (torch.cuda.stream(down) if cuda else _null_ctx()):
            hC.copy_(dC[:, :rows], non_blocking=cuda)
    if cuda:
        comp.synchronize()
        up.synchronize()
        down.synchronize()
    return launches


class _null_ctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class PeerBSlices:
    """B row-sliced across the ranks for the fused all-gather -> GEMM: rank r
    owns rows [cuts[r], cuts[r+1]) in a libmpfk device allocation exported
    with CUDA IPC; every rank maps every other rank's slice (NVLink peer
    memory), so one kernel per rank can pull the panels it needs while it
    computes (mpfk_gemm_device_pull).  The slices are the SURVEY's "each GPU
    uploads 1/G of B" layout (8(e)); nothing is broadcast."""

    def __init__(self, W: int, k: int, ld: int, group=None, align: int = 16):
        import torch.distributed as dist
        from . import linalg as L
        self.W, self.k, self.ld = W, k, ld
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.cuts = [shard_rows(k, world, r, align)[0] for r in range(world)] + [k]
        self.rank, self.world = rank, world
        self.rows = self.cuts[rank + 1] - self.cuts[rank]
        self.local = L.device_alloc(max(8 * W * self.rows * ld, 16))
        self._opened = []
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, L.ipc_handle(self.local), group=group)
            self.ptrs = []
            for r in range(world):
                if r == rank:
                    self.ptrs.append(self.local)
                else:
                    p = L.ipc_open(handles[r])
                    self._opened.append(p)
                    self.ptrs.append(p)
        else:
            self.ptrs = [self.local]

    def upload(self, host_planes):
        """host_planes: (W, rows, ld) float64 array of this rank's slice."""
        from . import linalg as L
        import numpy as np
        a = np.ascontiguousarray(host_planes, dtype=np.float64)
        assert a.shape == (self.W, self.rows, self.ld)
        if a.size:
            L.memcpy(self.local, a.ctypes.data, a.nbytes)

    def step(self, W, dA, dB, dC, rows, n, k, panel_rows=256, chunk_rows=2, stream=None, mode="pull",
             flags=0) -> int:
        """C_shard = A_shard * B with B gathered from the slices while the GEMM
        computes: mode "staged" -- the copy engines gather B in growing K
        panels and one GEMM launch per panel waits on that panel's event
        (mpfk_gemm_device_staged); mode "copy" -- the copy engines copy B's panels and
        flag them, the kernel waits per panel (mpfk_gemm_device_gathered);
        mode "pull" -- the GEMM's own CTAs pull the panels over peer memory
        (mpfk_gemm_device_pull)."""
        from . import linalg as L
        if rows == 0:
            return 0
        s = stream.cuda_stream if stream is not None else 0
        lda, ldb, ldc = dA.shape[2], dB.shape[2], dC.shape[2]
        if mode == "staged":
            return L.gemm_device_staged(W, rows, n, k, dA.data_ptr(), lda, dA.shape[1] * lda, dB.data_ptr(), ldb,
                                        dB.shape[1] * ldb, dC.data_ptr(), ldc, dC.shape[1] * ldc, self.ptrs,
                                        self.cuts, 0, s, flags)
        if flags:
            raise ValueError("PeerBSlices.step: flags (MPFK_LEAN) need mode 'staged'")
        if mode == "copy":
            return L.gemm_device_gathered(W, rows, n, k, dA.data_ptr(), lda, dA.shape[1] * lda, dB.data_ptr(), ldb,
                                          dB.shape[1] * ldb, dC.data_ptr(), ldc, dC.shape[1] * ldc, self.ptrs,
                                          self.cuts, panel_rows, s)
        if mode != "pull":
            raise ValueError("PeerBSlices.step: mode must be 'staged', 'copy' or 'pull'")
        return L.gemm_device_pull(W, rows, n, k, dA.data_ptr(), lda, dA.shape[1] * lda, dB.data_ptr(), ldb,
                                  dB.shape[1] * ldb, dC.data_ptr(), ldc, dC.shape[1] * ldc, self.ptrs, self.cuts,
                                  panel_rows, chunk_rows, s)

    def close(self):
        from . import linalg as L
        for p in self._opened:
            L.ipc_close(p)
        self._opened = []
        if self.local:
            L.device_free(self.local)
            self.local = 0


def gather_c(dC_shard, m: int, world: int, group=None, align: int = 64):
    """Assemble the replicated (W, m, ld) C from the row shards
    (all-gather); shards are padded to the common span length.  `align`
    must be the one the shards were cut with (shard_rows)."""
    import torch
    import torch.distributed as dist
    W, rows, ld = dC_shard.shape
    per = max(1, shard_rows(m, world, 0, align)[1])
    buf = torch.zeros((W, per, ld), dtype=dC_shard.dtype, device=dC_shard.device)
    buf[:, :rows] = dC_shard[:, :rows]
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf.contiguous(), group=group)
    spans = [shard_rows(m, world, r, align) for r in range(world)]
    out = torch.cat([p[:, : r1 - r0] for p, (r0, r1) in zip(parts, spans)], dim=1)
    return out.contiguous()
