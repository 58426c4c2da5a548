# quick iteration: TGN parity tests + launch list of a few bench steps
timeout 900 python -m pytest tests/test_tgn_gpu.py tests/test_eval_gpu.py -q --tb=short 2>&1 | grep -E "^E  |passed|failed|Error" | head -30
NTAIL=${NTAIL:-75} bash tools/gpu_ncu_list.sh
