# per-CTA phase stamps of several kernels of the C4 step: bash tools/gpu/run_phases.sh "2 4 6"
for pk in ${1:-2 4 6}; do
  make -B -j16 EXTRA="-DEKV_STAMPS -DEKV_PH_KERNEL=$pk" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
  echo "=== phase kernel $pk"; BOUNDS=${BOUNDS:-e4m3} timeout 300 python tools/trace.py 2>&1 | sed -n '/replay 2/,$p'
done
make -B -j16 all > /dev/null 2>&1
