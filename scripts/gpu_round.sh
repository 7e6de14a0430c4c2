# tests + bench sweep + ncu evidence for the current build
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
for w in dd1024 td1024 qd1024 dd8192 td4096 qd4096; do
  python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --out gpurun_out/bench_$w.json > gpurun_out/bench_$w.log 2>&1; echo bench $w rc=$?
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for w in dd8192 td4096 qd4096 dd1024; do
  python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/prof_plain_$w.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:mpgemm -c 1 --csv --log-file gpurun_out/metrics_$w.csv python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/ncu_m_$w.log 2>&1; echo ncu-metrics $w rc=$?
done
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ll_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dd8192.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ll.log 2>&1; echo ncu-launches rc=$?
python scripts/prof_gemm.py --workload dd8192 --launches 1 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mpgemm -c 1 -o gpurun_out/prof_dd8192 python scripts/prof_gemm.py --workload dd8192 --launches 1 > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?
