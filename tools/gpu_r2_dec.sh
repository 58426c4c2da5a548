# register-blocked decoder forward: parity tests (decoder-heavy subsets) + bench x2 + decoder ncu time
timeout 2400 python -m pytest tests -m gpu -x -q --tb=short -k "tgn or eval or bench_path" > gpurun_out/pytest_dec.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_dec.log
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --fp32-steps 0 --e2e-steps 5 > gpurun_out/bench_dec_$i.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_dec_$i.json'));print('dec',d['ms_per_step'],d['value'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_decoder -c 6 --csv --log-file gpurun_out/dec_ncu.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2>&1
grep -i "k_decoder" gpurun_out/dec_ncu.csv | awk -F'","' '{print $NF}' | head -6
