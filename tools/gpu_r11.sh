timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "newton" 2>&1 | grep -E "^E  |passed|failed" | head -20
