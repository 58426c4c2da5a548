# A/B of SPD_PREFETCH bits (GEMM weights 1, GRU weights 2, decoder W1 4) on the GDELT step
for m in 0 1 2 4 0 6; do
SPD_PREFETCH=$m timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 5 > gpurun_out/bench_knob_$m.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_knob_$m.json'));print('SPD_PREFETCH=$m',d['ms_per_step'],d['value'])"
done
