# Round profile: GPU tests, bench line, reference arm, in-graph trace, ncu launch list,
# ncu --set full of the top kernels, BASELINE configs 2/3/5 sweeps.
make -j4 all > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-200
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-120
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full > /dev/null 2>&1; echo ncu-list $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_score|k_attend_scores|k_topk|k_tau_sparse|k_delta_bar" -s 6 -c 5 -o gpurun_out/prof_full python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full > /dev/null 2>&1; echo ncu-full $?
timeout 900 python tools/sweeps.py all --out gpurun_out/sweeps.jsonl > /dev/null 2>&1; echo sweeps $?
bash tools/gpu/run_trace.sh 6 2>&1 | grep -A8 "replay 2" > gpurun_out/trace.txt; cat gpurun_out/trace.txt
