# parity tests, then the bench under each environment variant given as args
# (e.g. "SPD_UMMA_MAXBN=64"); prints one BENCH line per variant
timeout 900 python -m pytest tests -m gpu -q --tb=short -x 2>&1 | grep -E "^E  |passed|failed|Error" | head -30
for v in "" "$@"; do
  env $v timeout 600 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_sweep.json')); print('BENCH [$v]', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), d['roofline']['launch_ms'])" || tail -5 gpurun_out/bench_sweep.err
done
