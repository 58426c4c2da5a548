timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_tgn_gpu.py tests/test_bench_path_gpu.py -q -x --tb=short -k "gemm or tensor_core or bench_path or graph" 2>&1 | tail -3
for V in "SPD_UMMA_WIDE_BIG=0" "SPD_UMMA_WIDE_BIG=1" "SPD_UMMA_WIDE_BIG=0" "SPD_UMMA_WIDE_BIG=1"; do
  env $V timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 10 > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err
  python -c "import json;d=json.load(open('gpurun_out/bench_k.json'));p=d['phases_ms'];print('$V', d['ms_per_step'], p['gemm_qp'], p['gemm_dxbar'])"
done
