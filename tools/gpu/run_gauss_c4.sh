# Gaussian selector: GPU tests + the C4 (1M) Gaussian decode in the bench extras + C3 sweep point
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "gauss or Gauss" 2>&1 | tail -4
timeout 900 python bench.py --no-cpu-baseline --no-full > gpurun_out/bench_g.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/bench_g.log') if x.startswith('{')]
j=json.loads(l[-1]) if l else None
print('value', round(j['value'],1)); print('gauss', json.dumps(j.get('gaussian_selector')))" || tail -20 gpurun_out/bench_g.log
make -B -j16 EXTRA="-DEKV_STAMPS" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
echo "== C4 gauss trace"; timeout 300 python tools/trace.py $((1048576-200)) gauss 1 2>&1 | sed -n '/replay 2/,/per-CTA/p' | grep -v per-CTA
echo "== C3 gauss trace"; timeout 300 python tools/trace.py 131000 gauss 1 16 2>&1 | sed -n '/replay 2/,/per-CTA/p' | grep -v per-CTA
make -B -j16 all > /dev/null 2>&1
