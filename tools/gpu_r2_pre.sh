# parameter prefetch before the PDL wait (decoder, fused GRU, fwd/dgrad GEMMs): GPU suite, bench x3, timeline
timeout 2400 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_pre.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_pre.log
for i in 1 2 3; do
timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/bench_pre_$i.json 2> /dev/null; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_pre_$i.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'],d['roofline']['frac'])"
done
timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 --config reddit > gpurun_out/bench_pre_reddit.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_pre_reddit.json'));print('reddit',d['ms_per_step'],d['value'])"
timeout 900 python tools/trace_step.py > gpurun_out/timeline_pre.txt 2> /dev/null; rm -f gpurun_out/trace.json
head -3 gpurun_out/timeline_pre.txt
