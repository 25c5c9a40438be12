# Round profile: GPU tests, bench line, in-graph trace, ncu launch list and ncu --set full of the top kernels.
make -j4 all > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full > /dev/null 2>&1; echo ncu-list $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_score|k_attend_scores|k_topk|k_tau_sparse" -s 4 -c 4 -o gpurun_out/prof_full python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full > /dev/null 2>&1; echo ncu-full $?
bash tools/gpu/run_trace.sh 6 2>&1 | grep -A8 "replay 2" > gpurun_out/trace.txt; cat gpurun_out/trace.txt
