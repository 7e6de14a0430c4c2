# Round-2 final evidence in one call: GPU suite, smoke, acceptance gate,
# bit-parity and lean fuzz sweeps, both bench arms (driver-style arguments).
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/final_pytest_gpu.log
python __graft_entry__.py --smoke > gpurun_out/final_smoke.log 2>&1; echo smoke rc=$?
python tests/acceptance.py > gpurun_out/final_acceptance.log 2>&1; echo acceptance rc=$?; tail -3 gpurun_out/final_acceptance.log
python scripts/fuzz_parity.py 300 23 > gpurun_out/final_fuzz300.log 2>&1; echo fuzz rc=$?; tail -1 gpurun_out/final_fuzz300.log
python scripts/fuzz_lean.py 300 29 > gpurun_out/final_fuzz_lean.log 2>&1; echo fuzz_lean rc=$?; tail -1 gpurun_out/final_fuzz_lean.log
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench_reference.json 2> gpurun_out/final_bench_reference.err; echo reference rc=$?
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
