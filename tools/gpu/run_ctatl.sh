# per-CTA timeline of k_score (2) or k_attend_scores (1): bash tools/gpu/run_ctatl.sh <kid> <slot>
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_CTA_KERNEL=$1" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/cta_timeline.py "${@:2}" 2>&1 | tail -9
make -B -j16 all > /dev/null 2>&1
