mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_pull_gpu.py -q -x 2>&1 | tail -1
for cfg in "256 16" "256 4" "512 4" "128 2"; do set -- $cfg
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --workload dd8192 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --dist --fused-allgather --check --pull-panel $1 --pull-chunk $2 --out gpurun_out/bf.json > /dev/null 2>&1; echo "panel $1 chunk $2 rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bf.json')); print(d['value'], d['ms_per_step'], d['check_sharded_equals_one_shot'])"
done
