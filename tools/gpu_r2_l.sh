for V in 64 148 296 64 148 296; do
  SPD_GRU_WGRAD_CTAS=$V timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 10 > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err
  python -c "import json;d=json.load(open('gpurun_out/bench_l.json'));print('$V', d['ms_per_step'], d['phases_ms']['gru_bwd'])"
done
