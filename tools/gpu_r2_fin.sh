# fused finalize (split-K sums + time grads in Adam): parity tests + bench A/B
timeout 2400 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_fin.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_fin.log
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --steps 300 --fp32-steps 0 --e2e-steps 20 > gpurun_out/bench_fin_$i.json 2> /dev/null; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_fin_$i.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'])"
done
timeout 900 python tools/trace_step.py > gpurun_out/timeline_fin.txt 2> /dev/null; rm -f gpurun_out/trace.json
head -3 gpurun_out/timeline_fin.txt
