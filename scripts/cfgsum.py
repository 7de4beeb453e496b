import json,sys
tag=sys.argv[1]
for c in ("c1","c2","c3","c4","c5","paper","paper6"):
    try:
        d=json.loads(open(f'gpurun_out/{tag}_bench_{c}.log').read().strip().splitlines()[-1])
    except Exception as e:
        print(c,'ERR'); continue
    r=d['roofline']
    print(c, f"value {d['value']:.3e} step {d['ms_per_step']:.3f}ms frac {r['frac']:.3f} hbm {r.get('hbm',{}).get('frac',0):.3f} e2e {d['e2e']['value']:.3e} ({d['e2e']['ms_per_step']:.2f} ms) cpu {d.get('cpu_baseline',{}).get('value',0):.3e}")
