import json, sys
for f in sys.argv[1:]:
    print('==', f)
    for line in open(f):
        try:
            r = json.loads(line)
        except Exception:
            print(line.strip()[:200]); continue
        w = r['what']
        if w == 'sptrsv':
            print(f"{r.get('kernel','csr'):4s} bps={r['blocks_per_sm']} mask={r['sleep_ns']:4d}  L {r['lower_s']*1e3:7.3f} ms ({r['lower_frac']*100:4.1f}%, hop {r['hop_us_lower']:.2f}us)  U {r['upper_s']*1e3:7.3f} ms ({r['upper_frac']*100:4.1f}%, hop {r['hop_us_upper']:.2f}us)")
        else:
            print({k: (round(v, 5) if isinstance(v, float) else v) for k, v in r.items()})
