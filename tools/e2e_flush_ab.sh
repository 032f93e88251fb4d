for v in i32 u8 i32 u8; do
  if [ $v = u8 ]; then export NOLF_FLUSH_U8=1; else unset NOLF_FLUSH_U8; fi
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/e2ef.json 2>gpurun_out/e2ef.err
  python - "$v" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/e2ef.json').read().strip().splitlines()[-1])
print(sys.argv[1], round(d['ms_per_step'], 4), d['roofline']['kernel_ms']['k_march'], round(d['e2e']['value']), d['e2e'].get('device_us_per_step'))
PY
done
