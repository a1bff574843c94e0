timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r7_pytest.txt
timeout 400 python bench.py > gpurun_out/r7_bench.json 2> gpurun_out/r7_bench.err
python tools/sanitize_case.py > gpurun_out/r7_plain.txt 2>&1 && timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/r7_memcheck.txt 2>&1; echo memcheck_rc=$? >> gpurun_out/r7_memcheck.txt
cat gpurun_out/r7_pytest.txt; tail -3 gpurun_out/r7_memcheck.txt; python -c "
import json; d=json.load(open('gpurun_out/r7_bench.json')); print(d['value'], d['ms_per_step'], d['phases_ms_per_step'], d['roofline']['frac'], d['clocks'])"
