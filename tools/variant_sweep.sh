#!/bin/bash
# Build the library with each EXTRA flag set and print the bench phases (GPU box helper).
# usage: tools/variant_sweep.sh "<flags1>" "<flags2>" ...
for f in "$@"; do
  make -B EXTRA="$f" > /dev/null 2>&1 || { echo "BUILD FAILED: $f"; continue; }
  r=$(timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' | tail -1)
  echo "$f :: $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v,1) for k,v in d['phases_us'].items()}, 'full', round(d['full_entmax_us'],1))" 2>&1)"
done
make -B > /dev/null 2>&1
