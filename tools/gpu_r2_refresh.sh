# round-2 final evidence at the current state: default bench, reference arm,
# per-kernel ncu metrics of one step, ncu --set full of the attention / GRU /
# decoder kernels, CUPTI timeline; DyRep / JODIE benches
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/final_bench.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['roofline'],d['clocks'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --backbone jodie --no-cpu-baseline > gpurun_out/final_bench_jodie.json 2>/dev/null; echo "jodie rc=$?"
timeout 900 python bench.py --backbone dyrep --no-cpu-baseline > gpurun_out/final_bench_dyrep.json 2>/dev/null; echo "dyrep rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__registers_per_thread --clock-control none -c 600 --csv \
  --log-file gpurun_out/final_kernel_metrics.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> gpurun_out/final_ncu_metrics.err
python tools/kernel_table.py gpurun_out/final_kernel_metrics.csv > gpurun_out/final_kernel_table.txt; head -3 gpurun_out/final_kernel_table.txt; tail -1 gpurun_out/final_kernel_table.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_attn_abs_fwd|k_attn_abs_bwd|umma_gru|k_decoder" -s 8 -c 4 -o gpurun_out/final_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> gpurun_out/final_ncu_full.err
ncu -i gpurun_out/final_full.ncu-rep --page raw --csv > gpurun_out/ncu_k_attn_abs_raw.csv 2>/dev/null
ncu -i gpurun_out/final_full.ncu-rep --page details --csv > gpurun_out/ncu_final_details.csv 2>/dev/null
timeout 900 python tools/trace_step.py > gpurun_out/final_timeline.txt 2> gpurun_out/trace.err; rm -f gpurun_out/trace.json
head -3 gpurun_out/final_timeline.txt
ls -la gpurun_out/final_full.ncu-rep
