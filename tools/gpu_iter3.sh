# iterate: GPU parity tests, a short bench, a CUPTI timeline of one step
set -x
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K} 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --fp32-steps 50 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python tools/trace_step.py > gpurun_out/timeline.txt 2> gpurun_out/trace.err; rm -f gpurun_out/trace.json
tail -40 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err; head -80 gpurun_out/timeline.txt
