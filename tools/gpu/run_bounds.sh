# default bench line with extras (quality, budget sweep, Gaussian) for kv and e4m3 bounds
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for b in e4m3 kv; do
  timeout 900 python bench.py --no-cpu-baseline --no-full --bounds $b > gpurun_out/bench_$b.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/bench_$b.log') if x.startswith('{')]
j=json.loads(l[-1])
print('== $b value', round(j['value'],1), 'score', round(j['phases_us']['score_pages'],1), 'frac', round(j['roofline']['frac'],3))
for k in ['quality','recall_point','decode_only_us','decode_approx_tau']: print(k, j.get(k))
for x in j.get('budget_sweep') or []: print('  ', {k: (round(v,4) if isinstance(v,float) else v) for k,v in x.items() if k in ('budget','rho_pooled','rho_min','decode_us','speedup_vs_full_dense_v')})
g=j.get('gaussian_selector') or {}; print('gauss', {k:g.get(k) for k in ('rho_pooled','coverage','decode_us')})
"
done
