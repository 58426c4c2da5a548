# one full ncu capture of the named kernel(s) inside a short bench run; the
# report is exported to text pages on the box (the .ncu-rep is too big to ship)
K=${1:-k_attn_abs}
N=${2:-2}
OUT=${3:-gpurun_out/full}
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$K -c $N -f -o /tmp/ncu_full \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} \
  > gpurun_out/ncu_full_bench.json 2> gpurun_out/ncu_full_bench.err
ncu -i /tmp/ncu_full.ncu-rep --page details > ${OUT}_details.txt
ncu -i /tmp/ncu_full.ncu-rep --page raw --csv > ${OUT}_raw.csv
ncu -i /tmp/ncu_full.ncu-rep --page source --csv --print-source sass,cuda > ${OUT}_source.csv 2>/dev/null || \
  ncu -i /tmp/ncu_full.ncu-rep --page source --csv > ${OUT}_source.csv
gzip -9 -f ${OUT}_source.csv; ls -la gpurun_out/
