mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
python bench.py --out gpurun_out/bench_default.json > gpurun_out/bench_default.log 2>&1; echo bench rc=$?
python scripts/bench_ew.py > gpurun_out/bench_ew.jsonl 2>gpurun_out/bench_ew.err; echo ew rc=$?
for w in td4096 qd4096; do python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --out gpurun_out/bench_e2e_$w.json > /dev/null 2>&1; echo e2e $w rc=$?; done
