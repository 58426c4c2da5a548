# round-end style measurement: GPU tests, bench (ours + reference arm), ncu
# launch list + step table, ncu --set full of the attention kernels, CUPTI timeline
timeout 1200 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 1000 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
NTAIL=75 bash tools/gpu_ncu_list.sh > /dev/null
python tools/step_table.py gpurun_out/launches.csv 60 > gpurun_out/step_table.txt
bash tools/gpu_ncu_full.sh "k_attn_abs" 3 gpurun_out/ncu_k_attn_abs
timeout 900 python tools/trace_step.py > gpurun_out/timeline.txt 2> gpurun_out/trace.err; rm -f gpurun_out/trace.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/bench.json gpurun_out/bench_ref.json gpurun_out/smoke.log; head -3 gpurun_out/step_table.txt
