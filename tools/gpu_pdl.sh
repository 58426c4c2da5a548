# PDL on/off for the small-batch (B = 200) configs
for c in reddit lastfm; do
  for v in "" "SPD_PDL=1"; do
    env $v timeout 600 python bench.py --config $c --steps 500 --warmup 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/b.json 2> gpurun_out/b.err
    python -c "import json; d=json.load(open('gpurun_out/b.json')); print('$c [$v]', round(d['value']), d['ms_per_step'])" || tail -3 gpurun_out/b.err
  done
done
