PK=4
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=$PK" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/trace.py 2>&1 | tail -12
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=$PK -DEKV_ATT_PREF" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/trace.py 2>&1 | tail -12
