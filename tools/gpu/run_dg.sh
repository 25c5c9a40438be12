for n in 2 3 4; do
make -B -j16 EXTRA="-DEKV_DG_CTAS=$n" all > gpurun_out/build_v.log 2>&1 || { tail -5 gpurun_out/build_v.log; continue; }
echo "CTAS $n: $(timeout 600 python tools/sweeps.py c5 2>&1 | grep softmax | head -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['full_us'],1))")"
done
make -B -j16 all > /dev/null 2>&1
