# GPU suite + GDELT bench + small-batch configs
timeout 1500 python -m pytest tests -m gpu -q --tb=short 2>&1 | grep -E "^E  |passed|failed|Error" | head -30
timeout 900 python bench.py --steps 500 --warmup 5 --no-cpu-baseline --e2e-steps 20 > gpurun_out/b.json 2> gpurun_out/b.err
python -c "import json; d=json.load(open('gpurun_out/b.json')); print('gdelt', round(d['value']), d['ms_per_step'], round(d['e2e']['value']))" || tail -3 gpurun_out/b.err
for c in reddit lastfm ml25m; do
  timeout 600 python bench.py --config $c --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value']), d['ms_per_step'], round(d['e2e']['value']), d['device_memory_per_gpu'])" || tail -3 gpurun_out/bench_$c.err
done
