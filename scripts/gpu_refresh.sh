# refresh the judged evidence for the current build: bench lines (with e2e)
# of every BASELINE workload, the default line with the CPU baseline, ncu
# metric passes and --set full captures of the TD / QD GEMMs at full size
mkdir -p gpurun_out
for w in dd1024 td1024 qd1024 td4096 qd4096; do
  python bench.py --workload $w --no-cpu-baseline --out gpurun_out/bench_$w.json > gpurun_out/bench_$w.log 2>&1
  echo bench $w rc=$?
done
python bench.py --out gpurun_out/bench_default.json > gpurun_out/bench_default.log 2>&1; echo bench default rc=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for w in td4096 qd4096 td1024 qd1024; do
  ncu --metrics $M --clock-control none -k regex:mpgemm -c 1 --csv --log-file gpurun_out/metrics_$w.csv \
    python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/ncu_m_$w.log 2>&1; echo ncu-metrics $w rc=$?
done
for w in td4096 qd4096; do
  ncu --set full --clock-control none --import-source on -k regex:mpgemm -c 1 -o gpurun_out/prof_$w \
    python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/ncu_full_$w.log 2>&1
  echo ncu-full $w rc=$?
  ncu -i gpurun_out/prof_$w.ncu-rep --page raw --csv > gpurun_out/ncu_full_${w}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$w.ncu-rep --page details --csv > gpurun_out/ncu_full_${w}_details.csv 2>/dev/null
done
