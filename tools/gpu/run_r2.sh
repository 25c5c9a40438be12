# Round-2 check: build, GPU parity tests (incl. full-size), bench line, in-graph launch list.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/pytest_gpu.log 2>&1; tail -40 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -c 4000 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full --no-extras > /dev/null 2>&1; echo ncu $?
