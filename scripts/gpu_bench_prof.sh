# round-1 measurement: default bench (+e2e, +CPU baseline), reference arm,
# ncu launch list and one full capture per width.
mkdir -p gpurun_out
python bench.py --out gpurun_out/bench_default.json > gpurun_out/bench_default.log 2>&1; echo bench rc=$?
tail -c 3000 gpurun_out/bench_default.log
for w in td4096 qd4096; do python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo bench $w rc=$?; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo ref rc=$?
tail -c 1500 gpurun_out/bench_reference.log
python scripts/prof_gemm.py --workload dd8192 --launches 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dd8192.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo ncu-launches rc=$?
for w in dd8192 td4096 qd4096; do
  python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/prof_plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:mpgemm -c 1 -o gpurun_out/prof_$w python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/ncu_$w.log 2>&1; echo ncu $w rc=$?
done
ls -la gpurun_out
