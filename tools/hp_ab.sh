for c in 5 4; do for b in bench_old bench bench_old bench; do
  timeout 300 python $b.py --config $c --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/hp.json 2>gpurun_out/hp.err
  python - "$b" "$c" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/hp.json').read().strip().splitlines()[-1])
print(sys.argv[1], sys.argv[2], round(d['e2e']['value']), d['e2e']['host_us_per_step'], d['e2e']['device_us_per_step']['render'], d['verify'] if d.get('verify') is None else d['verify'].get('host_frame_bitwise_equal'))
PY
done; done
