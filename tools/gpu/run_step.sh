# build, GPU tests, bench headline (kv + e4m3), in-graph step trace (kv + e4m3)
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x ${PYTEST_K:-} 2>&1 | tail -4
TESTS= BENCHES="${BENCHES:---no-full --no-extras --no-cpu-baseline;--no-full --no-extras --no-cpu-baseline --bounds e4m3 --stats bf16}" bash tools/gpu/run_quick.sh 2>&1 | grep -v "^make"
make -B -j16 EXTRA="-DEKV_STAMPS" all > gpurun_out/build_st.log 2>&1 || tail -20 gpurun_out/build_st.log
for b in kv e4m3; do echo "=== trace $b"; BOUNDS=$b STATS=bf16 timeout 300 python tools/trace.py 2>&1 | grep -E "replay 2|start" | tail -9; done
make -B -j16 all > /dev/null 2>&1
