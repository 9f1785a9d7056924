import json,sys
for f in sys.argv[1:]:
    try:
        l=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], round(l['value'],1), round(l['ms_per_step']*1e3,1), {k: round(v*l['ms_per_step']*1e3,1) for k,v in l['kernel_share_of_step'].items()}, round(l['roofline']['achieved']), round(l['roofline']['frac'],3), (l.get('e2e') or {}).get('value'))
    except Exception as e: print(f, 'ERR', e, open(f).read()[-500:])
