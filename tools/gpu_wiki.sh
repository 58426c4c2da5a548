# full GPU suite, then the Wiki-shape AP/AUC test repeated with its printout
timeout 900 python -m pytest tests -m gpu -q --tb=short 2>&1 | grep -E "^E  |passed|failed|Error" | head -30
for i in 1 2; do
  timeout 600 python -m pytest tests/test_eval_gpu.py -q -s -k wiki_shape 2>&1 | grep -E "test AP|passed|failed"
done
