# final-state per-kernel evidence: ncu metrics table, ncu --set full (attention / GRU / decoder), CUPTI timeline
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__registers_per_thread --clock-control none -c 600 --csv \
  --log-file gpurun_out/f4_kernel_metrics.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> /dev/null
python tools/kernel_table.py gpurun_out/f4_kernel_metrics.csv > gpurun_out/f4_kernel_table.txt; head -1 gpurun_out/f4_kernel_table.txt; tail -1 gpurun_out/f4_kernel_table.txt
timeout 900 python tools/trace_step.py > gpurun_out/f4_timeline.txt 2> /dev/null; rm -f gpurun_out/trace.json; head -2 gpurun_out/f4_timeline.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_attn_abs_fwd|k_attn_abs_bwd|umma_gru|k_decoder" -s 8 -c 4 -o gpurun_out/f4_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> /dev/null
ncu -i gpurun_out/f4_full.ncu-rep --page raw --csv > gpurun_out/f4_ncu_raw.csv 2>/dev/null
ncu -i gpurun_out/f4_full.ncu-rep --page details --csv > gpurun_out/f4_ncu_details.csv 2>/dev/null
ls -la gpurun_out/f4_ncu_details.csv
