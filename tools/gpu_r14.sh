timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  |passed|failed|Error" | head -20
timeout 600 python bench.py --config cfg4 --events-per-rank 200 --no-cpu-baseline --e2e-steps 1 --steps 3 > gpurun_out/r14_bench_cfg4.json 2> gpurun_out/r14_bench_cfg4.err
tail -2 gpurun_out/r14_bench_cfg4.err; python -c "
import json; d=json.load(open('gpurun_out/r14_bench_cfg4.json')); print(d['value'], d['events_per_s'], d['ms_per_step'], d['phases_ms_per_step'], {k:(round(v['frac'],3), v['achieved']) for k,v in d['roofline_kernels'].items()})"
