make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_CTA_KERNEL=2" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
for b in kv e4m3; do echo "=== score_pages CTA timeline $b"; BOUNDS=$b timeout 300 python tools/cta_timeline.py 4 2>&1 | tail -9; done
