# round-2 checkpoint: full GPU suite, smoke, default bench, reference arm, N=2 functional, JODIE bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu_full.log 2>&1
tail -5 gpurun_out/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python -c "import json;d=json.load(open('gpurun_out/bench_full.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['roofline']['frac'],d['cpu_baseline']['value'] if d['cpu_baseline'] else None, d['clocks'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 300 gpurun_out/bench_ref.json
timeout 900 python bench.py --gpus 2 --config reddit --steps 50 --warmup 3 --no-cpu-baseline --fp32-steps 0 --e2e-steps 10 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
tail -c 400 gpurun_out/bench_n2.json; tail -3 gpurun_out/bench_n2.err
timeout 900 python bench.py --backbone jodie --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 10 --e2e-steps 20 > gpurun_out/bench_jodie.json 2> gpurun_out/bench_jodie.err
python -c "import json;d=json.load(open('gpurun_out/bench_jodie.json'));print('jodie', d['ms_per_step'],d['value'],d['e2e']['value'])"
