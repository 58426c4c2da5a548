timeout 1500 python -m pytest tests/test_tgn_gpu.py tests/test_bench_path_gpu.py tests/test_eval_gpu.py -q --tb=short -s 2>&1 | grep -E "test AP|passed|failed|FAILED|Error|assert" | tail -20
timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 10 --e2e-steps 10 > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
python -c "import json;d=json.load(open('gpurun_out/bench_d.json'));print(d['ms_per_step'],d['e2e']['value'])"
