# Round-end measurement set: default bench line (all extras), launch list of the timed step, ncu --set full of
# the step's kernels (traffic for the bench roofline), the full-baseline launch list, in-graph trace.
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/r2h_bench.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/r2h_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 40 --csv --log-file gpurun_out/r2h_launches_step.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full --no-extras > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_score|k_topk|k_attend_scores|k_tau_sparse|k_delta_bar|k_append" -s 6 -c 6 -f -o gpurun_out/r2h_step_full python tools/prof_kernel.py kv f32 decode 3 > gpurun_out/r2h_ncu.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"k_full_scores_mma|k_candidates|k_vstream" -c 3 -f -o gpurun_out/r2h_full_base python tools/full_only.py 1.5 > gpurun_out/r2h_ncu_full.log 2>&1; echo "ncu base rc=$?"
make -B -j16 EXTRA="-DEKV_STAMPS" all > gpurun_out/build_st.log 2>&1 && timeout 300 python tools/trace.py > gpurun_out/r2h_trace_step.txt 2>&1; make -B -j16 all > /dev/null 2>&1
tail -9 gpurun_out/r2h_trace_step.txt
