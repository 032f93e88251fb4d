for v in "" "--no-flush" "--e2e-mode copy" "--e2e-mode hostmap"; do
  timeout 300 python bench.py --no-cpu-baseline $v > gpurun_out/e2eab.json 2>gpurun_out/e2eab.err
  python - "$v" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/e2eab.json').read().strip().splitlines()[-1])
print(repr(sys.argv[1]), round(d['ms_per_step'], 4), round(d['e2e']['value']), d['e2e'].get('host_us_per_step'), d['e2e'].get('device_us_per_step'))
PY
done
