# SASS/source-level warp-stall sampling of one kernel: bash tools/gpu/run_ncu_src.sh <regex> <out>
make -j4 all > /dev/null 2>&1
timeout 600 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --warp-sampling-interval 0 --import-source on --clock-control none -k regex:"$1" -s 3 -c 1 -o gpurun_out/$2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full > /dev/null 2>&1; echo ncu $?
