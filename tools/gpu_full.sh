# round-end style measurement: GPU tests, bench (ours + reference arm), launch list, ncu full of the top kernel
set -x
timeout 900 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 300 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
NTAIL=75 bash tools/gpu_ncu_list.sh > /dev/null
python tools/step_table.py gpurun_out/launches.csv 60 > gpurun_out/step_table.txt
bash tools/gpu_ncu_full.sh k_attn_abs 2 gpurun_out/ncu_k_attn_abs
cat gpurun_out/pytest_gpu.log gpurun_out/bench.json gpurun_out/bench_ref.json
