# A/B the library variants in paper_2303_04086_b200/variants/ on one box:
# bench config per variant (kernel times, device step time); variants named
# stats* also dump the march work counters.
# usage: gpurun -- bash tools/ab.sh <prefix> [bench args...]
P=${1:-ab}; shift
for so in paper_2303_04086_b200/variants/libnolf_*.so; do
  n=$(basename $so .so); n=${n#libnolf_}
  case $n in stats*) export NOLF_STATS_DUMP=1;; *) unset NOLF_STATS_DUMP;; esac
  NOLF_LIB=$PWD/$so timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${P}_$n.json 2> gpurun_out/${P}_$n.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/${P}_$n.json').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()})" || tail -3 gpurun_out/${P}_$n.err
  grep STATS gpurun_out/${P}_$n.err
done
