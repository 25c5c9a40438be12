# build, a pytest subset (-k expression), bench value + in-graph trace of the C4 step
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "${1:-topk}" 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras --bounds ${BOUNDS:-kv} > gpurun_out/bench_q.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/bench_q.log') if x.startswith('{')]
j=json.loads(l[-1]) if l else None
print('value', round(j['value'],1) if j else open('gpurun_out/bench_q.log').read()[-1500:])"
make -B -j16 EXTRA="-DEKV_STAMPS" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
BOUNDS=${BOUNDS:-kv} timeout 300 python tools/trace.py 2>&1 | sed -n '/replay 2/,/per-CTA/p' | grep -v per-CTA
make -B -j16 all > /dev/null 2>&1
