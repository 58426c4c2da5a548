timeout 600 python -m pytest tests/test_tgn_gpu.py -q -x --tb=short -k "concurrent" 2>&1 | tail -3
timeout 1200 python bench.py --parts 2 --steps 200 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/gdelt_p2_seq.json 2> gpurun_out/gdelt_p2_seq.err
timeout 1200 python bench.py --parts 2 --concurrent --steps 200 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/gdelt_p2_conc.json 2> gpurun_out/gdelt_p2_conc.err
for f in gdelt_p2_seq gdelt_p2_conc; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['ms_per_step'], d['value'], d['e2e']['value'], d['device_memory_per_gpu'])" || tail -5 gpurun_out/$f.err; done
