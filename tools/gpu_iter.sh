# quick iteration: GPU parity tests + launch list of a few bench steps + a bench line
timeout 900 python -m pytest tests -m gpu -q --tb=short -x 2>&1 | grep -E "^E  |passed|failed|Error" | head -30
NTAIL=${NTAIL:-75} bash tools/gpu_ncu_list.sh > /dev/null
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('BENCH', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), d['gpu_launches'])"
