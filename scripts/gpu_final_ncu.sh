# ncu evidence at the round's final bit-exact kernels (TD 110 / QD 212 executed
# FP64 instructions per multiply-add): metric passes of the six workloads, full
# captures of DD 8192 and TD 4096, launch list of the device-timed bench steps
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for w in dd8192 td4096 qd4096 dd1024 td1024 qd1024; do
  python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/r02f_plain_$w.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:mpgemm -c 1 --csv --log-file gpurun_out/r02f_metrics_$w.csv python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/r02f_ncu_m_$w.log 2>&1; echo ncu-metrics $w rc=$?
done
for w in dd8192 td4096; do
  ncu --set full --clock-control none --import-source on -k regex:mpgemm -c 1 -o gpurun_out/r02f_full_$w python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/r02f_ncu_full_$w.log 2>&1; echo ncu-full $w rc=$?
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02f_ll_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02f_ncu_ll.log 2>&1; echo ncu-launches rc=$?
