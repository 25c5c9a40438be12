make -j4 all > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tau_pv|k_topk" -s 4 -c 2 -o gpurun_out/prof_tau python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full > /dev/null 2>&1; echo ncu $?
