import json, sys, csv, collections
f = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/bench.json'
try:
    j = json.loads(open(f).read().strip().splitlines()[-1])
    print('value %.0f req/s  us/step %.2f' % (j['value'], j['us_per_iteration']))
    r = j['roofline']; print(' roofline', {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()})
    print(' burst', j.get('burst_prefill'))
    print(' cpu', j['cpu_baseline'])
    print(' e2e', j['e2e'])
    print(' clocks', j['clocks'])
except Exception as e:
    print('bench parse error', e)
rows = list(csv.reader(open('gpurun_out/launches.csv')))
hdr = None; agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['Metric Name'] == 'gpu__time_duration.sum':
            agg[d['Kernel Name'][:50]].append(float(d['Metric Value']))
for k, v in agg.items(): print(f"  ncu {k:52s} n={len(v):4d} avg={sum(v)/len(v)/1e3:8.2f} us")
