# round-2 evidence: GPU suite, smoke, the driver's bench lines (both arms),
# the ncu launch list of the bench command and one --set full capture of
# the headline GEMM kernel.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/r02_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -12 gpurun_out/r02_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke rc=$?
S=$SECONDS; python bench.py --gpus 1 --steps 20 --warmup 5 --out gpurun_out/r02_bench.json > gpurun_out/r02_bench.log 2>&1; echo bench rc=$? wall $((SECONDS-S))
S=$SECONDS; python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 --out gpurun_out/r02_bench_reference.json > gpurun_out/r02_bench_reference.log 2>&1; echo ref rc=$? wall $((SECONDS-S))
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ll_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_ll.log 2>&1; echo ncu-launches rc=$?
python scripts/prof_gemm.py --workload dd8192 --launches 1 > gpurun_out/r02_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mpgemm -c 1 -o gpurun_out/r02_full_dd8192 python scripts/prof_gemm.py --workload dd8192 --launches 1 > gpurun_out/r02_ncu_full.log 2>&1; echo ncu-full rc=$?
