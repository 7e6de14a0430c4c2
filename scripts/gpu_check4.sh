mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_gpu.log
python -m paper_2101_06584_b200.mpfbench matmul --sizes 256,1024 --reps 3 --oracle-max 0 --out gpurun_out/mpfbench_matmul.csv 2> gpurun_out/mpfbench.err; echo mpfbench rc=$?
python -m paper_2101_06584_b200.mpfbench ewise --reps 3 --oracle-max 0 --out gpurun_out/mpfbench_ewise.csv 2>> gpurun_out/mpfbench.err; echo mpfbench-ew rc=$?
