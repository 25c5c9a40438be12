make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for b in kv e4m3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_score -s 2 -c 1 -f -o gpurun_out/prof_score_$b python tools/prof_kernel.py $b f32 score 3 > gpurun_out/ncu_$b.log 2>&1; echo "ncu $b rc=$?"
done
