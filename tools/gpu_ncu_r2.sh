# ncu --set full of one step's decoder, attention and tcgen05 GEMM launches
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_decoder|k_attn_abs|umma_gemm" -s 46 -c 23 \
  -o gpurun_out/step_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fp32-steps 0 > /dev/null 2> gpurun_out/ncu_step_full.err
tail -3 gpurun_out/ncu_step_full.err
ncu -i gpurun_out/step_full.ncu-rep --page raw --csv > gpurun_out/step_full_raw.csv 2>/dev/null
ls -la gpurun_out/step_full*
