timeout 900 python -m pytest tests/test_tgn_gpu.py -q --tb=short -k "device_shuffle or shuffle_combine" 2>&1 | tail -15
timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 10 --e2e-steps 50 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
python -c "import json;d=json.load(open('gpurun_out/bench_f.json'));print(d['ms_per_step'],d['e2e'])"
bash tools/gpu_configs_r2.sh 2>&1 | tail -14
