# iterate: GPU parity tests (-x), a short bench, the per-phase profile
set -x
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K} 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --fp32-steps 50 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -40 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
