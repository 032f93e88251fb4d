# Profile the config-4 march: work counters (stats build) + one ncu --set full capture of each hot kernel.
# usage: gpurun -- bash tools/prof.sh <prefix>
P=${1:-prof}
NOLF_STATS_DUMP=1 NOLF_LIB=$PWD/paper_2303_04086_b200/variants/libnolf_stats.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${P}_stats.json 2> gpurun_out/${P}_stats.err
grep STATS gpurun_out/${P}_stats.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${P}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_(cull_chunks|march_chunks|shade_tc|compose_live)" -c 4 -o gpurun_out/${P}_cfg4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${P}_ncu_full.log 2>&1
tail -2 gpurun_out/${P}_ncu_full.log
