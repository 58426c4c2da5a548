# re-entry check: full GPU suite, smoke, default bench, CUPTI timeline of one step
timeout 2400 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['roofline']['frac'],d['gpu_launches'],d['clocks'])"
timeout 900 python tools/trace_step.py > gpurun_out/timeline.txt 2> gpurun_out/trace.err; rm -f gpurun_out/trace.json
head -3 gpurun_out/timeline.txt
