mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -9 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()"; echo smoke rc=$?
python bench.py --out gpurun_out/bench_default.json > gpurun_out/bench_default.log 2>&1; echo bench rc=$?
for w in td4096 qd4096 dd1024; do python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --out gpurun_out/bench_$w.json > /dev/null 2>&1; echo bench $w rc=$?; done
