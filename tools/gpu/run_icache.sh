make -j4 all > /dev/null 2>&1
for cc in all none; do
timeout 300 ncu --metrics gpu__time_duration.sum --cache-control $cc --clock-control none --replay-mode kernel -k regex:"k_tau_sparse|k_delta_bar|k_topk|k_attend" -s 8 -c 8 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full 2>/dev/null | grep -E "gpu__time" | awk -F'","' '{print "'$cc'", $5, $NF}' | cut -c1-120
done
