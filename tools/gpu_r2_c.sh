# decoder fusion check: GPU tests (tgn + bench path + bridge), bench
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short -k "tgn or bench_path or bridge or eval or smoke" > gpurun_out/pytest_c.log 2>&1
tail -25 gpurun_out/pytest_c.log
timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 10 --e2e-steps 10 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
python -c "import json;d=json.load(open('gpurun_out/bench_c.json'));print(d['ms_per_step'],d['e2e']['value'],d['phases_ms'])"
timeout 900 python tools/trace_step.py > gpurun_out/timeline_c.txt 2> gpurun_out/trace.err; rm -f gpurun_out/trace.json
head -12 gpurun_out/timeline_c.txt
