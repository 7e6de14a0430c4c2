# e2e of the host path: copy-engine-gated single launch vs row-chunked launches
for w in ${@:-dd1024 td1024 qd1024 td4096 qd4096 dd8192}; do
  for mode in gated chunked; do
    if [ $mode = chunked ]; then export MPFK_CHUNKED_HOST=1; else unset MPFK_CHUNKED_HOST; fi
    python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --out gpurun_out/m_${w}_${mode}.json > /dev/null 2>&1
    python -c "import json;d=json.load(open('gpurun_out/m_${w}_${mode}.json'));e=d['e2e'];print('$w $mode', d['value'], e['value'], e.get('ms_breakdown'))"
  done
done
