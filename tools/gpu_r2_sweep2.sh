run() { env "$@" timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 5 > gpurun_out/sw.json 2> /dev/null; python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$*',d['ms_per_step'])"; }
run SPD_GRU_WGRAD_CTAS=32
run SPD_X=0
run SPD_GRU_WGRAD_CTAS=16
run SPD_GRU_WGRAD_CTAS=32 SPD_GRU_UB=16
run SPD_GRU_WGRAD_CTAS=48
run SPD_GRU_WGRAD_CTAS=32
