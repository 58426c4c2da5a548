# folded query x key projection: GPU suite, bench A/B (SPD_FOLD_Q=0 vs on)
timeout 2400 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_foldq.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_foldq.log
for m in 1 0 1 0; do
SPD_FOLD_Q=$m timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 5 > gpurun_out/bench_foldq_$m.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_foldq_$m.json'));print('SPD_FOLD_Q=$m',d['ms_per_step'],d['value'],d['gpu_launches'])"
done
