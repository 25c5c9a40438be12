# usage: bash tools/gpu/run_ph.sh <phase-kernel-id> [trace.py args]: in-graph trace + per-CTA phases
PK=$1; shift
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=$PK" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/trace.py "$@" 2>&1 | tail -14
