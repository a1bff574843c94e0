timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r5_pytest.txt
for v in variants/lib_s2.so paper_1709_08610_b200/libretina.so variants/lib_s8.so; do
  RETINA_LIB=$v timeout 300 python tools/variant_bench.py --events 1000 >> gpurun_out/r5_variants.jsonl 2>&1
done
timeout 400 python bench.py > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err
cat gpurun_out/r5_pytest.txt gpurun_out/r5_variants.jsonl; python -c "
import json; d=json.load(open('gpurun_out/r5_bench.json')); print(d['value'], d['ms_per_step'], d['phases_ms_per_step'], d['roofline']['frac'])"
