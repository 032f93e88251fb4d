for w in 0 96 100000; do
 for c in 4 5 3 1; do
  NOLF_COST_WAVES=$w timeout 300 python bench.py --config $c --steps 60 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/cw_${w}_$c.json 2>gpurun_out/cw_${w}_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/cw_${w}_$c.json').read().strip().splitlines()[-1]); print('waves $w cfg $c', round(d['ms_per_step'],4), d['launch']['march_order'], d['roofline']['kernel_ms'])"
 done
done
