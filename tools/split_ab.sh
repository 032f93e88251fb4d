# split march A/B: 1 GPU config 4, 4 GPUs configs 4 and 5
for sp in 1 2; do
  NOLF_MARCH_SPLIT=$sp python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/split_${sp}_n1.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/split_${sp}_n1.json').read().strip().splitlines()[-1]); print('split $sp n1 c4', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms']['k_march'],4))"
  for c in 4 5; do
    NOLF_MARCH_SPLIT=$sp timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29900 + c + sp)) bench.py --gpus 4 --config $c --no-e2e --verify > gpurun_out/split_${sp}_n4_c$c.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/split_${sp}_n4_c$c.json').read().strip().splitlines()[-1]); print('split $sp n4 c$c', round(d['ms_per_step'],4), d['verify']['bitwise_equal'], [round(r[0],4) for r in d['rank_kernel_ms']['ranks']])"
  done
done
