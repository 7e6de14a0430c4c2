# launch list of the bench's device-timed steps (the e2e legs use the
# copy-engine-gated host path, whose flag waits cannot progress under ncu's
# kernel serialisation) + a full capture of the DD n=1024 GEMM
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_ll_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_ncu_ll.log 2>&1; echo ncu-launches rc=$?
python scripts/prof_gemm.py --workload dd1024 --launches 1 > gpurun_out/r02_prof_dd1024.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mpgemm -c 1 -o gpurun_out/r02_full_dd1024 python scripts/prof_gemm.py --workload dd1024 --launches 1 > gpurun_out/r02_ncu_full_dd1024.log 2>&1; echo ncu-full rc=$?
S=$SECONDS; python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 --out gpurun_out/r02_bench_reference2.json > gpurun_out/r02_bench_reference2.log 2>&1; echo ref rc=$? wall $((SECONDS-S))
S=$SECONDS; python bench.py --gpus 1 --steps 20 --warmup 5 --out gpurun_out/r02_bench2.json > gpurun_out/r02_bench2.log 2>&1; echo bench rc=$? wall $((SECONDS-S))
