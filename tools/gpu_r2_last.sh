timeout 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/last_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/last_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/last_bench.json 2> gpurun_out/last_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/last_bench.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'],d['roofline']['frac'],d['clocks'])"
timeout 900 python tools/trace_step.py > gpurun_out/last_timeline.txt 2> /dev/null; rm -f gpurun_out/trace.json; head -2 gpurun_out/last_timeline.txt
