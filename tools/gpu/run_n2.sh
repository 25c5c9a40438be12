# N2 in-kernel collectives: device-mode sharded tests (virtual ranks + 2-process IPC) + the callback-mode tests
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sharded_dev.py -x -q 2>&1 | tail -25
timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_capacity.py -x -q 2>&1 | tail -3
