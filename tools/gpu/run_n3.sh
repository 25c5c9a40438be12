# N3 check: build, GPU tests (new fp8/bf16 metadata tests first), bench exact vs e4m3 bounds.
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_meta_fp8.py -q -x 2>&1 | tail -15
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(open(sys.argv[1]).read()[-2000:]); raise SystemExit
j=json.loads(l[-1])
print('value', round(j['value'],1), 'roofline', {k: j['roofline'][k] for k in ('achieved','frac','kernel_us','algorithmic_bytes_per_launch')}, 'phases', {k:round(v,1) for k,v in j['phases_us'].items()})
for k in ['quality','recall_point','decode_only_us','oracle_check','full_entmax_us','full_entmax_support_v_us']:
    print(' ',k, j.get(k))
for s in j.get('budget_sweep') or []: print('   sweep', {k:(round(v,4) if isinstance(v,float) else v) for k,v in s.items() if k in ('budget','rho_pooled','rho_min','decode_us','delta_mean')})
" $1; }
timeout 900 python bench.py --no-full > gpurun_out/bench_kv.log 2>&1; echo "=== bounds kv"; summ gpurun_out/bench_kv.log
timeout 900 python bench.py --no-full --bounds e4m3 --stats bf16 > gpurun_out/bench_e4m3.log 2>&1; echo "=== bounds e4m3"; summ gpurun_out/bench_e4m3.log
