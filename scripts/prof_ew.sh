mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_boundary_gpu.py tests/test_c_abi.py -q -x > gpurun_out/pytest_boundary.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_boundary.log
python scripts/bench_ew.py --n 16777216 --reps 3 > gpurun_out/ew_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:ew_kernel -c 7 --csv --log-file gpurun_out/metrics_ew.csv python scripts/bench_ew.py --n 16777216 --reps 3 > gpurun_out/ncu_ew.log 2>&1; echo ncu-ew rc=$?
