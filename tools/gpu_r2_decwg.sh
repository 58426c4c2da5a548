# A/B: decoder weight gradients forked after the dQ GEMM (SPD_DECWG_LATE=1) vs default
for m in 1 0 1 0; do
SPD_DECWG_LATE=$m timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 5 > gpurun_out/bench_decwg_$m.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_decwg_$m.json'));print('SPD_DECWG_LATE=$m',d['ms_per_step'],d['value'],d['gpu_launches'])"
done
