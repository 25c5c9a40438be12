make -B EXTRA=-DEKV_STAMPS all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/trace.py "$@" 2>&1 | tail -14
make -B all > /dev/null 2>&1
