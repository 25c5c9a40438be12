# Round-2 step anatomy: in-graph trace with top-k phases (PK=2) and tau phases (PK=6); per-CTA
# timelines of k_attend_scores (1) and k_score (2).
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=2" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
echo "=== trace, top-k phases"; timeout 300 python tools/trace.py 2>&1 | tail -16
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=6" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
echo "=== trace, tau phases"; timeout 300 python tools/trace.py 2>&1 | tail -12
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_CTA_KERNEL=1" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
echo "=== K-score CTA timeline"; timeout 300 python tools/cta_timeline.py 3 2>&1 | tail -9
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_CTA_KERNEL=2" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
echo "=== score_pages CTA timeline"; timeout 300 python tools/cta_timeline.py 4 2>&1 | tail -9
