# A/B of an environment knob on the C4 step: bash tools/gpu/run_ab_env.sh VAR "v1 v2" [bench args]
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
VAR=$1; VALS=$2; shift 2
for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras "$@" > gpurun_out/ab_$v.log 2>&1
  python -c "
import json,sys
l=[x for x in open('gpurun_out/ab_$v.log') if x.startswith('{')]
j=json.loads(l[-1]) if l else None
print('$VAR=$v', 'value', round(j['value'],1) if j else open('gpurun_out/ab_$v.log').read()[-1500:])"
done
make -B -j16 EXTRA="-DEKV_STAMPS" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
for v in $VALS; do echo "== trace $VAR=$v"; env $VAR=$v BOUNDS=${BOUNDS:-kv} timeout 300 python tools/trace.py 2>&1 | sed -n '/replay 2/,/per-CTA/p'; done
make -B -j16 all > /dev/null 2>&1
