# Round-end GPU check: gpu tests, smoke, bench lines for every BASELINE config + reference arm, ncu launch list and full capture.
# usage: gpurun --timeout 3000 -- bash tools/gpu_round.sh [prefix] [steps]   (outputs under gpurun_out/<prefix>_*)
# STEPS selects parts: t (pytest) s (smoke) b (bench cfg4) a (all configs) r (reference arm) n (ncu)
set -x
P=${1:-${P:-r02}}
STEPS=${2:-${STEPS:-tsbarn}}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
case $STEPS in *t*) timeout 1500 python -m pytest tests -m gpu -x -q -rf --durations=15 > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest_gpu.log;; esac
case $STEPS in *s*) timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${P}_smoke.log 2>&1;; esac
case $STEPS in *b*) timeout 600 python bench.py > gpurun_out/${P}_bench_cfg4.json 2> gpurun_out/${P}_bench_cfg4.err;; esac
case $STEPS in *a*) for c in 1 2 3 5; do timeout 400 python bench.py --config $c > gpurun_out/${P}_bench_cfg$c.json 2> gpurun_out/${P}_bench_cfg$c.err; done;; esac
case $STEPS in *r*) timeout 400 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err;; esac
case $STEPS in *n*)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${P}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_(cull_chunks|march_chunks|shade_tc|compose_live)" -s 12 -c 4 -o gpurun_out/${P}_cfg4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${P}_ncu_full.log 2>&1;;
esac
tail -5 gpurun_out/${P}_pytest_gpu.log; tail -2 gpurun_out/${P}_smoke.log; cat gpurun_out/${P}_bench_cfg4.json | head -c 3000
