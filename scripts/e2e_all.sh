# e2e leg (host buffers through the C ABI) of every BASELINE workload: value vs e2e
mkdir -p gpurun_out
for w in ${WORKLOADS:-dd1024 td1024 qd1024 td4096 qd4096 dd8192}; do
  python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --out gpurun_out/e_$w.json > gpurun_out/e_$w.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/e_$w.json'));e=d['e2e'];print('$w value', d['value'], 'e2e', e['value'], e['ms_breakdown'], e['matches_device_run'])"
done
