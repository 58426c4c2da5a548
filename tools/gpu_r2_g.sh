SPD_UMMA_DEEP=1 timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_bench_path_gpu.py -q --tb=short -x 2>&1 | tail -3
for V in "SPD_UMMA_DEEP=0" "SPD_UMMA_DEEP=1" "SPD_UMMA_MAXBN=128"; do
  env $V timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 10 > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err
  python -c "import json;d=json.load(open('gpurun_out/bench_g.json'));print('$V', d['ms_per_step'])"
done
SPD_UMMA_DEEP=1 timeout 900 python tools/trace_step.py > gpurun_out/timeline_g.txt 2> gpurun_out/trace.err; rm -f gpurun_out/trace.json
sed -n 1,75p gpurun_out/timeline_g.txt | awk '{printf "%s %s %s %s\n",$1,$2,$3,$4" "$5}'
