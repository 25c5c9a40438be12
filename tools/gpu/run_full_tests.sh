make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras 2>&1 | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['roofline']['kernel_us'])"
