for v in variants/*.so paper_1709_08610_b200/libretina.so; do
  RETINA_LIB=$v timeout 300 python tools/variant_bench.py --events 1000 >> gpurun_out/r6_variants.jsonl 2>&1
done
python -c "
import json
for l in open('gpurun_out/r6_variants.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(f\"{d['lib']:45s} grid {d['grid_ms']:7.2f} ms frac_fma {d['grid_frac_fma']:.3f} | ms {d['ms_ms']:7.2f} ms frac_mufu {d['ms_frac_mufu']:.3f}\")
"
