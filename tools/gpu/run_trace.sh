# usage: bash tools/gpu/run_trace.sh [phase-kernel-id] [trace.py args...]
PK=${1:-6}; shift
make -B EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=$PK" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/trace.py "$@" 2>&1 | tail -16
make -B all > /dev/null 2>&1
