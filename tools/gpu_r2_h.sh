timeout 1200 python -m pytest tests/test_tgn_gpu.py -q --tb=short -x 2>&1 | tail -25
