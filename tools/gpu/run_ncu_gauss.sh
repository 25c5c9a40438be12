# full GPU suite, then source-level stall sampling of k_gauss_select on the C3 (16 x 128K) workload
make -j4 all > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section Occupancy --warp-sampling-interval 0 --import-source on --clock-control none -k regex:k_gauss -c 1 -o gpurun_out/gauss_src python tools/trace.py 131000 gauss 1 16 > /dev/null 2>&1; echo ncu $?
