"""One rank of the CPU launcher test (tests/test_launch.py): started by
paper_2101_06584_b200.launch.spawn_local_ranks -- the launcher bench.py
--gpus N uses -- with RANK / WORLD_SIZE / MASTER_* in the environment.  Joins a
gloo group, computes its row shard of C = A*B with the oracle as compute
(the GPU box has one GPU), and rank 0 checks the assembled C bit for bit
against the one-shot product, printing one JSON line.

  python tests/launch_worker.py W m k n [fail_rank]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2101_06584_b200.dist import gather_c, shard_rows, sharded_gemm_step

    W, m, k, n = (int(x) for x in sys.argv[1:5])
    fail_rank = int(sys.argv[5]) if len(sys.argv) > 5 else -1
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    if rank == fail_rank:
        sys.exit(3)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ld = (n + 3) & ~3
        # every rank generates only its own rows of A (the BASELINE generator
        # addresses rows directly, like bench.py's fill_baseline(row0=...))
        r0, r1 = shard_rows(m, world, rank, align=8)
        rows = r1 - r0
        A = O.orc_fill_baseline(W, rows, k, 1, wide=W > 2, row0=r0)
        dA = torch.from_numpy(A)
        dB = torch.zeros((W, k, ld), dtype=torch.float64)
        if rank == 0:
            dB.copy_(torch.from_numpy(O.orc_fill_baseline(W, k, n, 2, wide=W > 2)))
        dC = torch.zeros((W, max(rows, 1), ld), dtype=torch.float64)

        def oracle_gemm(W_, dA_, dB_, dC_, rows_, n_, k_, ld_):
            dC_[:, :rows_] = torch.from_numpy(O.orc_gemm(dA_.numpy(), dB_.numpy(), k_, n_))
            return 1

        launches = sharded_gemm_step(W, dA, dB, dC, rows, n, k, ld, gemm=oracle_gemm)
        Cfull = gather_c(dC[:, :rows], m, world, align=8)
        if rank == 0:
            want = O.orc_gemm(O.orc_fill_baseline(W, m, k, 1, wide=W > 2),
                              O.orc_fill_baseline(W, k, n, 2, wide=W > 2), k, n)
            same = bool(np.array_equal(Cfull.numpy().view(np.uint64), want.view(np.uint64)))
            print(json.dumps({"nranks": dist.get_world_size(), "backend": dist.get_backend(),
                              "check_sharded_equals_one_shot": same, "launches": launches}), flush=True)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
