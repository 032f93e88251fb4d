for sp in 1 2 1 2; do for c in 4 5; do
  NOLF_MARCH_SPLIT=$sp timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/msp.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/msp.json').read().strip().splitlines()[-1]); print('split $sp cfg $c', round(d['ms_per_step'],4), d['roofline']['kernel_ms']['k_march'])"
done; done
