# build the library with each EXTRA variant (';'-separated in VARIANTS) and time the bench headline
IFS=';' read -ra VS <<< "$VARIANTS"
for x in "${VS[@]}"; do
  make -B -j16 EXTRA="$x" all > gpurun_out/build_v.log 2>&1 || { echo "build failed: $x"; tail -5 gpurun_out/build_v.log; continue; }
  timeout 600 python bench.py ${BENCH_ARGS:---no-full --no-extras --no-cpu-baseline} > gpurun_out/bench_v.log 2>&1
  echo "== $x"; python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(open(sys.argv[1]).read()[-1500:]); raise SystemExit
j=json.loads(l[-1]); print('value', round(j['value'],1), 'score_us', round(j['roofline']['kernel_us'],1), 'GB/s', round(j['roofline']['achieved']), 'phases', {k:round(v,1) for k,v in j['phases_us'].items()})
" gpurun_out/bench_v.log
done
