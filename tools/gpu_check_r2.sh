# round-2 check: full GPU test suite (no -x), smoke, short bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --tb=short ${PYTEST_K} > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --fp32-steps 50 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -30 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
