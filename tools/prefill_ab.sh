for pf in state on; do for c in 4 5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + c)) bench.py --gpus 4 --config $c --verify --prefill $pf --no-e2e > gpurun_out/pf_${pf}_c$c.json 2> gpurun_out/pf_${pf}_c$c.err
  python -c "import json; d=json.loads(open('gpurun_out/pf_${pf}_c$c.json').read().strip().splitlines()[-1]); print('$pf', $c, round(d['ms_per_step'],4), round(d['value']), d['verify'].get('bitwise_equal'), [[round(x,4) for x in r[:3]] for r in d['rank_kernel_ms']['ranks']])" || tail -3 gpurun_out/pf_${pf}_c$c.err
done; done
