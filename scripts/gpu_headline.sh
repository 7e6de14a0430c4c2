mkdir -p gpurun_out
S=$SECONDS; python bench.py --out gpurun_out/bench_default.json > gpurun_out/bench_default.log 2>&1; echo bench rc=$? wall $((SECONDS-S)) s; tail -1 gpurun_out/bench_default.log
S=$SECONDS; python bench.py --impl reference --out gpurun_out/bench_reference.json > gpurun_out/bench_reference.log 2>&1; echo ref rc=$? wall $((SECONDS-S)) s; tail -1 gpurun_out/bench_reference.log
