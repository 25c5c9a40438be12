# a5 full-cache baseline: parity tests + C4 timings of every variant + a launch list
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "full or prop2 or softmax" 2>&1 | tail -5
timeout 300 python tools/full_only.py 1.5
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"^k_" -c 12 --csv --log-file gpurun_out/full_launches.csv python tools/full_only.py 1.5 > /dev/null 2>&1; echo ncu $?
