timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  |passed|failed|Error" | head -20
for v in variants/lib_s3_*.so paper_1709_08610_b200/libretina.so; do
  RETINA_LIB=$v timeout 300 python tools/variant_bench.py --config cfg4 --events 100 >> gpurun_out/r15_variants.jsonl 2>&1
done
python -c "
import json
for l in open('gpurun_out/r15_variants.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(f\"{d['lib']:45s} grid {d['grid_ms']:7.2f} ms frac_fma {d['grid_frac_fma']:.3f} | ms {d['ms_ms']:7.2f} ms frac_mufu {d['ms_frac_mufu']:.3f}\")
"
timeout 600 python bench.py --config cfg4 --events-per-rank 200 --no-cpu-baseline --e2e-steps 1 --steps 3 > gpurun_out/r15_bench_cfg4.json 2> gpurun_out/r15_bench_cfg4.err
timeout 400 python bench.py > gpurun_out/r15_bench.json 2> gpurun_out/r15_bench.err
python -c "
import json
for f in ('gpurun_out/r15_bench_cfg4.json','gpurun_out/r15_bench.json'):
    d=json.load(open(f)); print(f, d['value'], d['events_per_s'], d['ms_per_step'], d['phases_ms_per_step'], {k:(round(v['frac'],3), v['achieved']) for k,v in d['roofline_kernels'].items()})"
