# final headline-kernel evidence (paired B columns): metric pass + full capture of DD 8192 and DD 1024
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for w in dd8192 dd1024; do
  python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/r02d_plain_$w.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:mpgemm -c 1 --csv --log-file gpurun_out/r02d_metrics_$w.csv python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/r02d_ncu_m_$w.log 2>&1; echo ncu-metrics $w rc=$?
  ncu --set full --clock-control none --import-source on -k regex:mpgemm -c 1 -o gpurun_out/r02d_full_$w python scripts/prof_gemm.py --workload $w --launches 1 > gpurun_out/r02d_ncu_full_$w.log 2>&1; echo ncu-full $w rc=$?
done
