# bench.py's N > 1 path on the one GPU: 2 ranks on cuda:0 (gloo for the NCCL-mode collectives)
make -j16 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
EKV_SAME_DEVICE=1 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-full --no-extras --n ${N:-262144} > gpurun_out/bench_n2.log 2>&1; echo rc=$?
python -c "
import json
l=[x for x in open('gpurun_out/bench_n2.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench_n2.log').read()[-3000:]); raise SystemExit
j=json.loads(l[-1]); print('value',j['value'],j['config']['parallelism']); print(json.dumps(j.get('seq_sharded'),indent=1))"
