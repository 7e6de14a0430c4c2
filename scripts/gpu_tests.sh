mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/pytest_gpu.log
timeout 120 ./tests/_build/shim_parity 97 > gpurun_out/shim_parity.log 2>&1; echo shim rc=$?
cat gpurun_out/shim_parity.log
