# compute-sanitizer over small steps of every C-ABI path: memcheck, racecheck, synccheck, initcheck
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
python tools/sanitize_step.py > /dev/null 2>&1   # warm (first import)
for tool in memcheck synccheck initcheck racecheck; do
  echo "== $tool"
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_step.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|OK$|Error|error" gpurun_out/sanitize_$tool.log | head -8
done
