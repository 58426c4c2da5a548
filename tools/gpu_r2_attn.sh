# branch-free attention slots + vectorised Adam finalize: full GPU suite, bench x2, timeline, attention ncu times
timeout 2400 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_attn.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_attn.log
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/bench_attn_$i.json 2> /dev/null; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_attn_$i.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'],d['roofline']['frac'],d['roofline']['other_kernels_ms'])"
done
timeout 900 python tools/trace_step.py > gpurun_out/timeline_attn.txt 2> /dev/null; rm -f gpurun_out/trace.json
head -3 gpurun_out/timeline_attn.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_attn_abs_fwd|k_attn_abs_bwd|k_adam" -s 6 -c 3 -o gpurun_out/attn_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> gpurun_out/attn_ncu.err
ncu -i gpurun_out/attn_full.ncu-rep --page details --csv > gpurun_out/ncu_attn_details.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/ncu_attn_details.csv | grep -E "==|Duration|Ipc|Occupancy|Registers"
