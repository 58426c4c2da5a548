timeout 1200 python -m pytest tests/test_tgn_gpu.py tests/test_eval_gpu.py -q -x --tb=short 2>&1 | tail -3
mkdir -p gpurun_out/cfgc
for P in 2 4 8; do
  timeout 600 python bench.py --config reddit --parts $P --concurrent --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/cfgc/reddit_p${P}_conc.json 2> gpurun_out/cfgc/reddit_p${P}_conc.err
done
for K in 0 0.05 0.1; do
  timeout 600 python bench.py --config lastfm --parts 4 --hub-k $K --concurrent --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/cfgc/lastfm_p4_k${K}_conc.json 2> gpurun_out/cfgc/lastfm_p4_k${K}_conc.err
done
for P in 2 4 8; do
  timeout 900 python bench.py --config ml25m --parts $P --concurrent --steps 200 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/cfgc/ml25m_p${P}_conc.json 2> gpurun_out/cfgc/ml25m_p${P}_conc.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/cfgc/*.json")):
    try:
        d = json.load(open(f)); c = d["config"]
        print(f"{f.split('/')[-1]:28s} P={c['partitions']} k={c['hub_k']} {d['value']/1e6:7.3f} M/s {d['ms_per_step']:.4f} ms/step e2e {d['e2e']['value']/1e6:7.3f} M/s sync={d.get('epoch_end_sync_ms', 0):.2f} ms")
    except Exception as ex:
        print(f, "ERR", ex, open(f.replace('.json','.err')).read()[-400:])
PY
