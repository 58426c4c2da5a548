timeout 1200 python -m pytest tests/test_tgn_gpu.py -m gpu -x -q --tb=short -k "fold_variants" > gpurun_out/pytest_foldvar.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_foldvar.log
