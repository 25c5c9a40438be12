make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for t in 0 1 2 0; do echo "== EKV_DBG_TWICE=$t"; EKV_DBG_TWICE=$t timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras 2>&1 | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'])"; done
