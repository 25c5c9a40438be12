# tau-kernel candidate capacity sweep: in-graph timelines for C4 (1M top-k) and C3 (16 x 128K Gaussian)
make -B EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=6" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
for cap in 0 4096 2048; do
  echo "== cap $cap C4"; EKV_TS_CAP=$cap timeout 300 python tools/trace.py 2>&1 | sed -n "/replay 2/,\$p"
  echo "== cap $cap C3"; EKV_TS_CAP=$cap timeout 300 python tools/trace.py 131000 gauss 1 16 2>&1 | sed -n "/replay 2/,\$p"
done
make -B all > /dev/null 2>&1
