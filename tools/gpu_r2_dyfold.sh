timeout 2400 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_dyfold.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_dyfold.log
timeout 900 python bench.py --backbone dyrep --no-cpu-baseline --fp32-steps 0 > gpurun_out/bench_dyfold.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_dyfold.json'));print('dyrep',d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'])"
timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 > gpurun_out/bench_tgnfold.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_tgnfold.json'));print('tgn',d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'],d['roofline']['frac'])"
