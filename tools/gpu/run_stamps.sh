# Phase stamps of top-k / tau kernels (library built with -DEKV_STAMPS), then the normal build.
make -B EXTRA=-DEKV_STAMPS all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/stamps.py 2>&1 | grep -E "^tau|^topk|clock"
timeout 300 python tools/cand_count.py 2>&1 | tail -5
make -B all > /dev/null 2>&1
