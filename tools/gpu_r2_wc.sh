timeout 2400 python -m pytest tests -m gpu -x -q --tb=short -k "tgn or eval or bench_path or multirank" > gpurun_out/pytest_wc.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_wc.log
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 5 > gpurun_out/bench_wc_$i.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_wc_$i.json'));print('wc',d['ms_per_step'],d['value'],d['gpu_launches'])"
done
