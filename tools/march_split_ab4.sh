for sp in 1 2 1 2; do for c in 4 5; do
  NOLF_MARCH_SPLIT=$sp timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29610 + sp + c)) bench.py --gpus 4 --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/msp4.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/msp4.json').read().strip().splitlines()[-1]); print('split $sp cfg $c', round(d['ms_per_step'],4), [r[0] for r in d['rank_kernel_ms']['ranks']])"
done; done
