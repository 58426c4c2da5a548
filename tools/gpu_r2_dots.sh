# grouped guard-free dots: GPU suite, bench x2, attention ncu durations + instruction counts
timeout 2400 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_dots.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_dots.log
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/bench_dots_$i.json 2> /dev/null; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_dots_$i.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'],d['roofline']['frac'],d['roofline']['other_kernels_ms'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_attn_abs_fwd|k_attn_abs_bwd|k_adam" -s 6 -c 3 -o gpurun_out/dots_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> gpurun_out/dots_ncu.err
ncu -i gpurun_out/dots_full.ncu-rep --page details --csv > gpurun_out/ncu_dots_details.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/ncu_dots_details.csv | grep -E "==|Duration|Ipc|Occupancy"
