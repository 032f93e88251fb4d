# A/B the marcher's live-chunk order on one box: spatial, heaviest-first by
# candidate count, heaviest-first by the previous frame's measured durations.
# usage: gpurun [--gpus N] -- bash tools/order_ab.sh <prefix> <gpus> [bench args...]
P=${1:-ord}; G=${2:-1}; shift 2
run() {  # name, extra args
  if [ "$G" = 1 ]; then timeout 400 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e "${@:2}" > gpurun_out/${P}_$1.json 2> gpurun_out/${P}_$1.err
  else timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $G --steps 100 --warmup 10 --no-cpu-baseline --no-e2e "${@:2}" > gpurun_out/${P}_$1.json 2> gpurun_out/${P}_$1.err; fi
  python -c "import json; d=json.loads(open('gpurun_out/${P}_$1.json').read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],4), d['rank_kernel_ms']['ranks'])" || tail -3 gpurun_out/${P}_$1.err
}
run spatial --march-order spatial "$@"
run heavy_cnt --march-order heavy --chunk-cost 0 "$@"
run heavy_cost --march-order heavy --chunk-cost 1 "$@"
run auto "$@"
