make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for N in 512 1024 512 1024; do echo "NT $N"; EKV_TOPK_NT=$N timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras 2>&1 | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['phases_us'])"; done
timeout 900 python -m pytest tests -m gpu -q -x -k "topk or decode or fullsize or certified" 2>&1 | tail -2
