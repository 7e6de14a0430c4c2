mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
for w in dd8192 td4096 qd4096 dd1024; do python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --out gpurun_out/bench_e2e_$w.json > gpurun_out/bench_e2e_$w.log 2>&1; echo e2e $w rc=$?; done
