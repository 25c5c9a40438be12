# quick: build, a test selection (TESTS), bench headline lines for the given bench arg sets (BENCHES, ';'-separated)
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
[ -n "$TESTS" ] && timeout 1200 python -m pytest $TESTS -q -x 2>&1 | tail -4
IFS=';' read -ra BS <<< "${BENCHES:---no-full --no-extras --no-cpu-baseline}"
i=0
for a in "${BS[@]}"; do i=$((i+1)); timeout 900 python bench.py $a > gpurun_out/bench_q$i.log 2>&1; echo "== $a"; python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(open(sys.argv[1]).read()[-1500:]); raise SystemExit
j=json.loads(l[-1]); print('value', round(j['value'],1), 'score_us', round(j['roofline']['kernel_us'],1), 'GB/s', round(j['roofline']['achieved']), 'frac', round(j['roofline']['frac'],3), 'phases', {k:round(v,1) for k,v in j['phases_us'].items()})
for k in ('quality','recall_point','decode_only_us','full_entmax_us','full_entmax_support_v_us','full_entmax_dense_v_frac','gaussian_selector','oracle_check'):
    if j.get(k) is not None: print('  ', k, j[k])
" gpurun_out/bench_q$i.log; done
