# top-k phase trace + quick bench (current tree)
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --no-cpu-baseline --no-full --no-extras > gpurun_out/bench_q.log 2>&1; tail -c 1500 gpurun_out/bench_q.log
make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=2" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
timeout 300 python tools/trace.py 2>&1 | tail -22
