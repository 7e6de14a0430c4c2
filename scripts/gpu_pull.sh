mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_bench_dist_gpu.py -q -x > gpurun_out/pytest_dist.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_dist.log
for w in dd8192 qd4096; do
  python bench.py --workload $w --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --out gpurun_out/b_plain_$w.json > /dev/null 2>&1; echo plain $w rc=$?
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --workload $w --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --dist --fused-allgather --check --out gpurun_out/b_fused_$w.json > gpurun_out/b_fused_$w.log 2>&1; echo fused $w rc=$?
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --workload $w --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --dist --check --out gpurun_out/b_nccl_$w.json > gpurun_out/b_nccl_$w.log 2>&1; echo nccl $w rc=$?
done
