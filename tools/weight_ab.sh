# rank-0 weight sweep on N GPUs (configs 4 and 5, --verify)
N=${1:-4}
for w in 1.0 0.9 0.8; do for c in 4 5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29800 + c)) bench.py --gpus $N --config $c --verify --rank0-weight $w --no-e2e > gpurun_out/w_${w}_c$c.json 2> gpurun_out/w_${w}_c$c.err
  python -c "import json; d=json.loads(open('gpurun_out/w_${w}_c$c.json').read().strip().splitlines()[-1]); print('$w', $c, round(d['ms_per_step'],4), round(d['value']), d['verify'].get('bitwise_equal'), [[round(x,4) for x in r[:3]] for r in d['rank_kernel_ms']['ranks']])" || tail -3 gpurun_out/w_${w}_c$c.err
done; done
