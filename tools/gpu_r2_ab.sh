# A/B: fused head on/off; reference arm; launch lists
for FH in 0 1; do
SPD_FUSED_HEAD=$FH timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 10 --e2e-steps 10 > gpurun_out/bench_fh$FH.json 2> gpurun_out/bench_fh$FH.err
SPD_FUSED_HEAD=$FH bash tools/gpu_ncu_list.sh gpurun_out/launches_fh$FH.csv > /dev/null
python tools/step_table.py gpurun_out/launches_fh$FH.csv 70 > gpurun_out/step_table_fh$FH.txt
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for FH in 0 1; do python -c "import json;d=json.load(open('gpurun_out/bench_fh$FH.json'));print($FH,d['ms_per_step'],d['e2e']['value'])"; head -4 gpurun_out/step_table_fh$FH.txt; done
cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
