# round-2 final evidence (current state): GPU suite, smoke, default bench, reference arm, backbones,
# per-kernel ncu metrics, ncu --set full of attention / GRU / decoder, CUPTI timeline
timeout 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/f3_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f3_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/f3_bench.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'],d['roofline']['frac'],d['clocks'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f3_bench_ref.json 2> /dev/null; echo "ref rc=$?"
timeout 900 python bench.py --backbone jodie --no-cpu-baseline > gpurun_out/f3_bench_jodie.json 2>/dev/null; echo "jodie rc=$?"
timeout 900 python bench.py --backbone dyrep --no-cpu-baseline > gpurun_out/f3_bench_dyrep.json 2>/dev/null; echo "dyrep rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__registers_per_thread --clock-control none -c 600 --csv \
  --log-file gpurun_out/f3_kernel_metrics.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> /dev/null
python tools/kernel_table.py gpurun_out/f3_kernel_metrics.csv > gpurun_out/f3_kernel_table.txt; head -2 gpurun_out/f3_kernel_table.txt; tail -1 gpurun_out/f3_kernel_table.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_attn_abs_fwd|k_attn_abs_bwd|umma_gru|k_decoder" -s 8 -c 4 -o gpurun_out/f3_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> /dev/null
ncu -i gpurun_out/f3_full.ncu-rep --page raw --csv > gpurun_out/f3_ncu_raw.csv 2>/dev/null
ncu -i gpurun_out/f3_full.ncu-rep --page details --csv > gpurun_out/f3_ncu_details.csv 2>/dev/null
timeout 900 python tools/trace_step.py > gpurun_out/f3_timeline.txt 2> /dev/null; rm -f gpurun_out/trace.json
head -3 gpurun_out/f3_timeline.txt
