# BASELINE configs at P > 1 on one GPU (partitions as local workers of one trainer):
# Reddit SEP 1/2/4/8, LastFM shared-hub sweep k in {0, .01, .05, .10} at P = 4, ML25M P = 1/2/4/8
mkdir -p gpurun_out/cfg
for P in 1 2 4 8; do
  timeout 600 python bench.py --config reddit --parts $P --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/cfg/reddit_p$P.json 2> gpurun_out/cfg/reddit_p$P.err
done
for K in 0 0.01 0.05 0.1; do
  timeout 600 python bench.py --config lastfm --parts 4 --hub-k $K --steps 300 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/cfg/lastfm_p4_k$K.json 2> gpurun_out/cfg/lastfm_p4_k$K.err
done
for P in 1 2 4 8; do
  timeout 900 python bench.py --config ml25m --parts $P --steps 200 --warmup 5 --no-cpu-baseline --fp32-steps 0 --e2e-steps 20 > gpurun_out/cfg/ml25m_p$P.json 2> gpurun_out/cfg/ml25m_p$P.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/cfg/*.json")):
    try:
        d = json.load(open(f))
        c = d["config"]
        print(f"{f.split('/')[-1]:24s} P={c['partitions']} k={c['hub_k']} {d['value']/1e6:7.3f} M/s {d['ms_per_step']:.4f} ms/step e2e {d['e2e']['value']/1e6:7.3f} M/s shared={d.get('shared_hubs')} sync={d.get('epoch_end_sync_ms', 0):.2f} ms mem={d['device_memory_per_gpu']}")
    except Exception as ex:
        print(f, "ERR", ex)
PY
