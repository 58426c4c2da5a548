# iterate: selected GPU tests (PYTEST_K), bench (BENCH_ARGS), CUPTI timeline of one step
set -x
if [ -n "${PYTEST_K}" ]; then timeout 1500 python -m pytest tests -m gpu -x -q --tb=short -k "${PYTEST_K}" > gpurun_out/pytest_it.log 2>&1; fi
timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 10 --e2e-steps 10 ${BENCH_ARGS} > gpurun_out/bench_it.json 2> gpurun_out/bench_it.err
timeout 900 python tools/trace_step.py > gpurun_out/timeline_it.txt 2> gpurun_out/trace.err; rm -f gpurun_out/trace.json
set +x
tail -5 gpurun_out/pytest_it.log
python -c "import json;d=json.load(open('gpurun_out/bench_it.json'));print(d['ms_per_step'],d['e2e']['value'],d['phases_ms'])"
tail -3 gpurun_out/bench_it.err
sed -n 1,100p gpurun_out/timeline_it.txt | awk '{printf "%s %s %s %s\n",$1,$2,$3,$4" "$5}'
