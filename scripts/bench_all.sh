# device-resident bench of every BASELINE workload (no e2e / CPU baseline)
mkdir -p gpurun_out
for w in ${WORKLOADS:-dd1024 td1024 qd1024 dd8192 td4096 qd4096}; do
  python bench.py --workload $w --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e \
    --out gpurun_out/bench_$w.json > gpurun_out/bench_$w.log 2>&1
  python - "$w" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_{sys.argv[1]}.json"))
r = d["roofline"]
print(f"{sys.argv[1]:8s} value {d['value']:9.2f} kernel_ms {r['kernel_ms']:9.3f} frac {r['frac']:.4f} clocks {d['clocks']['sm_mhz']}")
PY
done
