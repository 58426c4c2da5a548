timeout 1500 python -m pytest tests -m gpu -x -q --tb=short -k "tgn or bench_path or eval" 2>&1 | tail -3
timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err
python -c "import json;d=json.load(open('gpurun_out/bench_i.json'));print(d['ms_per_step'],d['e2e']['value'])"
timeout 1500 python tools/shuffle_timing.py gdelt 2 > gpurun_out/shuffle_timing_gdelt.json 2> gpurun_out/shuffle_timing.err
cat gpurun_out/shuffle_timing_gdelt.json; tail -4 gpurun_out/shuffle_timing.err
