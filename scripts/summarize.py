import json, csv, collections, sys
for f in ['gpurun_out/bench_fast.log','gpurun_out/plain.log']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "value %.3e"%d['value'], "ms/step %.2f"%d['ms_per_step'], "tr_ms %.1f"%d['roofline']['transport_ms'], "e2e %.3e"%d['e2e']['value'], d.get('cpu_baseline',{}).get('value'))
    except Exception as e: print(f, open(f).read()[-800:])
rows=list(csv.reader(open('gpurun_out/launches_fast.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
seq=[]; agg=collections.Counter()
for r in rows[hi+1:]:
    if len(r)<=vi: continue
    v=float(r[vi].replace(',',''))/1e3
    agg[r[ki][:50]]+=v
    if 'k_fast_segment' in r[ki] or 'low_order' in r[ki]:
        seq.append(('SEG' if 'fast' in r[ki] else 'LO', v))
print(' '.join("%s:%.0f"%s for s in seq[:48]))
for k,v in agg.most_common(8): print("%10.0f us %s"%(v,k))
