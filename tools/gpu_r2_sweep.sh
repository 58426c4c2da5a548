# knob sweep at the final state (one bench each, 300 steps)
run() { env "$@" timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 5 > gpurun_out/sw.json 2> /dev/null; python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$*',d['ms_per_step'])"; }
run SPD_X=0
run SPD_DHPULL_CTAS=296
run SPD_TATTN_CTAS=148
run SPD_GRU_WGRAD_CTAS=128
run SPD_GRU_UB=16
run SPD_X=0
run SPD_DHPULL_CTAS=222
run SPD_GRU_WGRAD_CTAS=32
