# ncu --set full with source of the decode step's top-k, K-score and tau kernels (C4, e4m3 bounds)
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_topk|k_attend_scores|k_tau_sparse|k_delta_bar" -s 8 -c 4 -f -o gpurun_out/prof_sel python tools/prof_kernel.py ${BOUNDS:-e4m3} f32 decode 5 > gpurun_out/ncu_sel.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_sel.log
