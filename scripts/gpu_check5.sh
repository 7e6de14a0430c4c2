mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bench_dist_gpu.py -q -x > gpurun_out/pytest_dist.log 2>&1; echo pytest-dist rc=$?; tail -15 gpurun_out/pytest_dist.log
python scripts/tune.py --sizes 1024,4096 --reps 2 > gpurun_out/tune2.log 2>&1; echo tune rc=$?
