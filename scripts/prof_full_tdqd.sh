# ncu --set full captures of the TD and QD GEMMs (n=2048: same tiles and
# per-CTA behaviour as the 4096 configs, a quarter of the replay time)
mkdir -p gpurun_out
for w in td4096 qd4096; do
  python scripts/prof_gemm.py --workload $w --n 2048 --launches 1 > gpurun_out/prof_plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:mpgemm -c 1 -o gpurun_out/prof_$w \
    python scripts/prof_gemm.py --workload $w --n 2048 --launches 1 > gpurun_out/ncu_full_$w.log 2>&1
  echo ncu-full $w rc=$?
done
