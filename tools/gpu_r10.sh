timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r10_pytest.txt
tail -30 gpurun_out/r10_pytest.txt
