timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r12_pytest.txt
timeout 400 python bench.py > gpurun_out/r12_bench.json 2> gpurun_out/r12_bench.err
timeout 300 python bench.py --update newton --no-cpu-baseline --e2e-steps 1 > gpurun_out/r12_bench_newton.json 2> gpurun_out/r12_bench_newton.err
timeout 300 python tools/cost_constants.py > gpurun_out/r12_cost.json 2>&1
cat gpurun_out/r12_pytest.txt gpurun_out/r12_cost.json; tail -2 gpurun_out/r12_bench_newton.err
python -c "
import json
for f in ('gpurun_out/r12_bench.json','gpurun_out/r12_bench_newton.json'):
    d=json.load(open(f)); print(f, d['value'], d['events_per_s'], d['ms_per_step'], d['phases_ms_per_step'], {k:round(v['frac'],3) for k,v in d['roofline_kernels'].items()})"
