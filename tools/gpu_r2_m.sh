SPD_PDL_MAIN=1 timeout 600 python -m pytest tests/test_tgn_gpu.py -q -x --tb=short -k "graph or tensor_core or steps_match" 2>&1 | tail -2
for V in "SPD_PDL_MAIN=0" "SPD_PDL_MAIN=1" "SPD_PDL_MAIN=0" "SPD_PDL_MAIN=1"; do
  env $V timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 10 > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err
  python -c "import json;d=json.load(open('gpurun_out/bench_m.json'));print('$V', d['ms_per_step'])"
done
for V in "SPD_PDL_MAIN=0" "SPD_PDL_MAIN=1"; do
  env $V SPD_PDL=0 timeout 900 python bench.py --config reddit --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 10 > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err
  python -c "import json;d=json.load(open('gpurun_out/bench_m.json'));print('reddit pdl-off', '$V', d['ms_per_step'])"
done
timeout 900 python bench.py --config reddit --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 10 > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err
python -c "import json;d=json.load(open('gpurun_out/bench_m.json'));print('reddit default (pdl all)', d['ms_per_step'])"
