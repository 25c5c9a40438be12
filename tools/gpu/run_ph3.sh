PK=4
for X in "-DEKV_ATT_SLEEP=5000" "-DEKV_MBAR_HINT=2000"; do
echo "=== $X"
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=$PK $X" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/trace.py 2>&1 | grep -A9 per-CTA
done
