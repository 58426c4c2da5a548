SPD_GRU_UB=16 timeout 900 python -m pytest tests/test_tgn_gpu.py tests/test_bench_path_gpu.py -q -x --tb=short -k "tensor_core or bench_path or graph" 2>&1 | tail -3
for V in "SPD_GRU_UB=32" "SPD_GRU_UB=16" "SPD_GRU_UB=32" "SPD_GRU_UB=16"; do
  env $V timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 10 > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err
  python -c "import json;d=json.load(open('gpurun_out/bench_j.json'));print('$V', d['ms_per_step'], d['phases_ms']['gru_fwd'])"
done
