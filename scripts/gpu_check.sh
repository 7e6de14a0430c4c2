mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
lscpu | grep -E 'Model name|^CPU\(s\)|Thread|Flags' | cut -c1-150
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
for w in dd1024 td1024 qd1024 dd8192; do timeout 300 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -2; done > gpurun_out/bench_quick.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
