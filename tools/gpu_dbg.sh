timeout 1200 python -m pytest tests/test_tgn_gpu.py -q --tb=short 2>&1 | grep -E "^E  |passed|failed|Error|^tests" | head -60
