make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "topk or decode or fullsize or certified or edges" 2>&1 | tail -2
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras 2>&1 | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['phases_us'])"; done
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=2" all > gpurun_out/build_st.log 2>&1; timeout 300 python tools/trace.py 2>&1 | tail -20; make -B -j16 all > /dev/null 2>&1
