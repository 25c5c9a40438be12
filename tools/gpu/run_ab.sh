# A/B: current tree vs build/ab_prev (an older commit's tree): bench line + in-graph trace.
R=$PWD
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(open(sys.argv[1]).read()[-2000:]); raise SystemExit
j=json.loads(l[-1])
print('value', round(j['value'],1), 'roofline', round(j['roofline']['frac'],3), 'phases', {k:round(v,1) for k,v in j['phases_us'].items()})
for k in ['quality','recall_point','decode_only_us','gaussian_selector','oracle_check']:
    print(' ',k, j.get(k))
" $1; }
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --no-cpu-baseline --no-full ${BENCH_ARGS:-} > gpurun_out/bench_cur.log 2>&1; echo "=== current"; summ gpurun_out/bench_cur.log
cd build/ab_prev && timeout 900 python bench.py --no-cpu-baseline --no-full ${BENCH_ARGS:-} > $R/gpurun_out/bench_prev.log 2>&1; cd $R; echo "=== prev"; summ gpurun_out/bench_prev.log
make -B -j16 EXTRA="-DEKV_STAMPS" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
echo "=== trace current"; timeout 300 python tools/trace.py 2>&1 | tail -12
cd build/ab_prev && make -B -j16 EXTRA="-DEKV_STAMPS" all > /dev/null 2>&1; echo "=== trace prev"; timeout 300 python tools/trace.py 2>&1 | tail -12
