# bench lines for the other BASELINE configs at P = 1 (device memory footprint included)
for c in reddit lastfm ml25m; do
  timeout 900 python bench.py --config $c --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value']), d['ms_per_step'], round(d['e2e']['value']), d['device_memory_per_gpu'])" || tail -3 gpurun_out/bench_$c.err
done
