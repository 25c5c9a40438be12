# A/B over build flags x env settings on the C4 step (bench value + in-graph trace):
#   bash tools/gpu/run_ab_build.sh "-DEKV_EF=0|-DEKV_EF=1" "EKV_TOPK_PREFETCH=0|EKV_TOPK_PREFETCH=1"
IFS='|' read -ra BUILDS <<< "$1"; IFS='|' read -ra ENVS <<< "${2:-X=0}"; shift 2
for bf in "${BUILDS[@]}"; do
  make -B -j16 EXTRA="$bf" all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
  for ev in "${ENVS[@]}"; do
    env $ev timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras "$@" > gpurun_out/ab.log 2>&1
    python -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')]
j=json.loads(l[-1]) if l else None
print('[$bf] [$ev]', 'value', round(j['value'],1) if j else open('gpurun_out/ab.log').read()[-1500:])"
  done
  make -B -j16 EXTRA="$bf -DEKV_STAMPS" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
  for ev in "${ENVS[@]}"; do echo "== trace [$bf] [$ev]"; env $ev BOUNDS=${BOUNDS:-kv} timeout 300 python tools/trace.py 2>&1 | sed -n '/replay 2/,/per-CTA/p' | grep -v per-CTA; done
done
make -B -j16 all > /dev/null 2>&1
