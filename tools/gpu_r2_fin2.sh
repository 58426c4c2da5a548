timeout 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/fin2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fin2_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/fin2_bench.json 2> gpurun_out/fin2_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/fin2_bench.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'],d['roofline']['frac'],d['clocks'])"
