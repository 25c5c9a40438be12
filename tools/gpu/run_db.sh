make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras 2>&1 | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['roofline']['kernel_us'])"
make -B -j16 EXTRA="-DEKV_STAMPS" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/trace.py 2>&1 | tail -8
make -B -j16 all > /dev/null 2>&1
