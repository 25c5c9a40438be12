# e4m3 box-kernel occupancy variants: CTAs per SM x pages per stage
for V in "2 16" "3 8" "3 12" "3 10"; do set -- $V
make -B -j16 EXTRA="-DEKV_SCORE_E4M3_CTAS=$1 -DEKV_SCORE_E4M3_SP=$2" all > gpurun_out/build_v.log 2>&1 || { tail -5 gpurun_out/build_v.log; continue; }
grep -A2 "k_scoreI13__nv_bfloat16Li4ELi1ELi1E" build_ptxas.log | grep -o "[0-9]* bytes spill stores" | head -1
echo "CTAS $1 SP $2: $(timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras --bounds e4m3 2>&1 | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['roofline']['kernel_us'])")"
done
make -B -j16 all > /dev/null 2>&1
