# multirank peer test; timeline; per-kernel ncu metric table; ncu full of umma gemm
timeout 900 python -m pytest tests/test_multirank_gpu.py -x -q --tb=short > gpurun_out/pytest_multirank.log 2>&1
tail -15 gpurun_out/pytest_multirank.log
timeout 900 python tools/trace_step.py > gpurun_out/timeline.txt 2> gpurun_out/trace.err; rm -f gpurun_out/trace.json
head -80 gpurun_out/timeline.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__registers_per_thread --clock-control none -c 600 --csv \
  --log-file gpurun_out/kernel_metrics.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> gpurun_out/ncu_metrics.err
tail -3 gpurun_out/ncu_metrics.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_gemm_kernel -s 400 -c 6 -o gpurun_out/umma_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> gpurun_out/ncu_full.err
tail -3 gpurun_out/ncu_full.err
