timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k tensor 2>&1 | tail -25 > gpurun_out/r8_tensor.txt
cat gpurun_out/r8_tensor.txt
timeout 300 python tools/variant_bench.py --events 1000 --algo 3 > gpurun_out/r8_tc_bench.json 2>&1; cat gpurun_out/r8_tc_bench.json
