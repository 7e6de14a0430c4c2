mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
python -m paper_2101_06584_b200.mpfbench matmul --sizes 256,1024,4096 --precision dd,qd --algo block,strassen --reps 2 --oracle-max 0 --out gpurun_out/mpfbench_strassen.csv 2> gpurun_out/mpfbench.err; echo mpfbench rc=$?
python -m paper_2101_06584_b200.mpfbench matmul --sizes 8192 --precision dd --algo block,strassen --cutoff 1024 --reps 1 --oracle-max 0 --out gpurun_out/mpfbench_strassen8k.csv 2>> gpurun_out/mpfbench.err; echo mpfbench8k rc=$?
