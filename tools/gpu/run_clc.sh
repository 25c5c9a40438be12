make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for T in 0 10 15 25; do echo "tail $T"; EKV_SCORE_TAIL=$T timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras 2>&1 | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['roofline']['kernel_us'], j['roofline']['frac'])"; done
EKV_SCORE_TAIL=15 timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras --bounds e4m3 2>&1 | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('e4m3', j['value'], j['roofline']['kernel_us'], j['roofline']['frac'])"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
