rm -f gpurun_out/r13_variants.jsonl
for v in variants/*.so paper_1709_08610_b200/libretina.so; do
  RETINA_LIB=$v timeout 300 python tools/variant_bench.py --events 1000 >> gpurun_out/r13_variants.jsonl 2>&1
done
python -c "
import json
for l in open('gpurun_out/r13_variants.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(f\"{d['lib']:45s} ms {d['ms_ms']:7.2f} ms frac_mufu {d['ms_frac_mufu']:.3f}\")
"
