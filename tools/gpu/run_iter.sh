# Iteration check: GPU tests, bench line, in-graph trace (top-k phases).
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; python -c "
import json
l=[x for x in open('gpurun_out/bench.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench.log').read()[-3000:]); raise SystemExit
j=json.loads(l[-1])
print('value', j['value'], 'roofline', round(j['roofline']['frac'],3), 'phases', j['phases_us'])
for k in ['full_entmax_us','full_entmax_support_v_us','e2e','e2e_eager','oracle_check','cpu_baseline','quality','recall_point','decode_only_us']:
    print(k, j.get(k))
"
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=${PK:-2}" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/trace.py 2>&1 | tail -16
