# State of the C4 step: bench lines (kv / e4m3 bounds), in-graph traces, ncu full of e4m3 k_score
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(open(sys.argv[1]).read()[-2000:]); raise SystemExit
j=json.loads(l[-1])
print('value', round(j['value'],1), 'roofline', round(j['roofline']['frac'],3), 'phases', {k:round(v,1) for k,v in j['phases_us'].items()})
" $1; }
for b in kv e4m3; do
  timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras --bounds $b > gpurun_out/bench_$b.log 2>&1; echo "== bench $b"; summ gpurun_out/bench_$b.log
done
make -B -j16 EXTRA="-DEKV_STAMPS" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
for b in kv e4m3; do echo "== trace $b"; BOUNDS=$b timeout 300 python tools/trace.py 2>&1 | sed -n '/replay 2/,/per-CTA/p'; done
make -B -j16 all > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_score -s 2 -c 1 -f -o gpurun_out/prof_score_e4m3 python tools/prof_kernel.py e4m3 f32 score 3 > gpurun_out/ncu_e4m3.log 2>&1; echo "ncu rc=$?"
