import cProfile, pstats, sys, os
sys.argv = ["train_bench.py", "--steps", "200"]
sys.path.insert(0, "/root/repo/tools")
import train_bench
cProfile.run("train_bench.main()", "/tmp/tp.pstats")
pstats.Stats("/tmp/tp.pstats").sort_stats("tottime").print_stats(18)
