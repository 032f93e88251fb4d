# Multi-GPU bench lines (configs 4 and 5, --verify) on the GPUs of one box.
# usage: gpurun --gpus N -- bash tools/scale.sh <prefix> "<gpu counts>"
P=${1:-scale}; NS=${2:-"2 4"}
for n in $NS; do for c in 4 5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n * 10 + c)) bench.py --gpus $n --config $c --verify > gpurun_out/${P}_n${n}_c$c.json 2> gpurun_out/${P}_n${n}_c$c.err
  python -c "import json; d=json.loads(open('gpurun_out/${P}_n${n}_c$c.json').read().strip().splitlines()[-1]); print($n, $c, round(d['ms_per_step'],4), round(d['value']), round(d['e2e']['value']), d['verify'].get('bitwise_equal'), d['verify'].get('host_frame_bitwise_equal'), d['rank_kernel_ms']['ranks'])" || tail -3 gpurun_out/${P}_n${n}_c$c.err
done; done
