rm -f gpurun_out/r17_variants.jsonl
for v in variants/lib_s3_*.so paper_1709_08610_b200/libretina.so; do
  RETINA_LIB=$v timeout 300 python tools/variant_bench.py --config cfg4 --events 100 >> gpurun_out/r17_variants.jsonl 2>&1
done
python -c "
import json
for l in open('gpurun_out/r17_variants.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(f\"{d['lib']:45s} ms {d['ms_ms']:7.2f} ms frac_mufu {d['ms_frac_mufu']:.3f}\")
"
