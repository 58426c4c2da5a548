timeout 1500 python -m pytest tests/test_tgn_gpu.py tests/test_bench_path_gpu.py tests/test_eval_gpu.py tests/test_gemm_gpu.py -q --tb=short -s 2>&1 | grep -E "test AP|passed|failed|FAILED|Error|assert|errors" | tail -20
timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 10 --e2e-steps 10 > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
python -c "import json;d=json.load(open('gpurun_out/bench_e.json'));print(d['ms_per_step'],d['e2e']['value'],d['phases_ms'])"
tail -3 gpurun_out/bench_e.err
SPD_GRU_FUSED=0 timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 10 > gpurun_out/bench_e0.json 2> gpurun_out/bench_e0.err
python -c "import json;d=json.load(open('gpurun_out/bench_e0.json'));print('unfused GRU', d['ms_per_step'])"
timeout 900 python tools/trace_step.py > gpurun_out/timeline_e.txt 2> gpurun_out/trace.err; rm -f gpurun_out/trace.json
sed -n 1,30p gpurun_out/timeline_e.txt | awk '{printf "%s %s %s %s\n",$1,$2,$3,$4" "$5}'
