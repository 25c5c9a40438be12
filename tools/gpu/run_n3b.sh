make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_meta_fp8.py -q -x 2>&1 | tail -5
for b in kv e4m3; do timeout 600 python bench.py --no-full --no-extras --no-cpu-baseline --bounds $b --stats bf16 > gpurun_out/bench_$b.log 2>&1; echo "== $b"; python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
j=json.loads(l[-1]); print('value', round(j['value'],1), 'score_us', round(j['roofline']['kernel_us'],1), 'GB/s', round(j['roofline']['achieved']), 'frac', round(j['roofline']['frac'],3))
" gpurun_out/bench_$b.log; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_score -s 2 -c 1 -f -o gpurun_out/prof_score_e4m3 python tools/prof_kernel.py e4m3 f32 score 3 > gpurun_out/ncu_e4m3.log 2>&1; echo "ncu rc=$?"
