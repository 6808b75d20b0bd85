"""Print sweep JSONL files compactly: pattern window d us/seq-layer frac_of_bound."""
import json, sys
for f in sys.argv[1:]:
    print("==", f)
    for l in open(f):
        try:
            d = json.loads(l)
        except Exception:
            print("  ", l.strip()[:160]); continue
        print(f"  {d['pattern']:9s} {str(d['window']):4s} d={d.get('d', 64):2d} {d['us_per_seq_layer']:7.2f} us  {d['frac_of_bound']:.3f} ({d['bound']})")
