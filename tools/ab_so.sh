# A/B two builds of libspeed_b200.so on one box: ab/old.so vs ab/new.so, alternating
L=paper_2308_14129_b200/libspeed_b200.so
for c in ${AB_CONFIGS:-gdelt}; do for r in 1 2; do for v in old new; do
  cp ab/$v.so $L
  timeout 600 python bench.py --config $c --steps 400 --warmup 5 --no-cpu-baseline --fp32-steps 2 --e2e-steps 2 ${BENCH_ARGS} 2>/dev/null \
    | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c $v',d['ms_per_step'],d['phases_ms'].get('head_fwd'),d['clocks']['sm_mhz'])"
done; done; done
