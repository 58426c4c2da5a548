timeout 1500 python -m pytest tests -m gpu -x -q --tb=short -k "jodie_backbone or concurrent_workers or eval_scores" > gpurun_out/pytest_dyrep.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_dyrep.log
timeout 900 python bench.py --backbone dyrep --no-cpu-baseline > gpurun_out/bench_dyrep.json 2> gpurun_out/bench_dyrep.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_dyrep.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'])"
tail -3 gpurun_out/bench_dyrep.err
