# A/B --split 2 (two interleaved tile halves on two streams) on G GPUs, configs 4 and 5.
# usage: gpurun [--gpus G] -- bash tools/split2_ab.sh <prefix> <G>
P=${1:-sp}; G=${2:-1}
for c in 4 5; do for sp in 1 2; do
  if [ "$G" = 1 ]; then timeout 400 python bench.py --config $c --split $sp --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/${P}_c${c}_s$sp.json 2> gpurun_out/${P}_c${c}_s$sp.err
  else timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $((29550 + c + sp)) bench.py --gpus $G --config $c --split $sp --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --verify > gpurun_out/${P}_c${c}_s$sp.json 2> gpurun_out/${P}_c${c}_s$sp.err; fi
  python -c "import json; d=json.loads(open('gpurun_out/${P}_c${c}_s$sp.json').read().strip().splitlines()[-1]); print('cfg $c split $sp', round(d['ms_per_step'],4), (d.get('verify') or {}).get('bitwise_equal'), [r[:3] + [r[4]] for r in d['rank_kernel_ms']['ranks']][:2])" || tail -3 gpurun_out/${P}_c${c}_s$sp.err
done; done
