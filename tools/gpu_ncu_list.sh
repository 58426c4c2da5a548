# per-kernel launch list of a few bench steps (times are cold-cache, serialised)
OUT=${1:-gpurun_out/launches.csv}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none ${NCU_EXTRA} -c ${NCU_COUNT:-700} --csv \
  --log-file $OUT python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/ncu_bench.json 2> gpurun_out/ncu_bench.err
python tools/launch_table.py $OUT | tail -${NTAIL:-80}
