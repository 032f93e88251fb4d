"""Summarise an ncu capture (+ launch list) into profiles/<name>.md / .json.

usage: python tools/ncu_summary.py gpurun_out/r01_prof.ncu-rep [gpurun_out/r01_launches.csv] profiles/r01
"""

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_B",
    "dram__bytes_write.sum": "dram_write_B",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}
    per = defaultdict(list)
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        d = {}
        for k, lab in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    d[lab] = float(v) * scale.get(units[i], 1)
                except ValueError:
                    pass
        per[name.split("(")[0].replace("void ", "")].append(d)
    return per


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            break
    h = rows[i]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[i + 1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")))
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v) / 1e3} for k, v in d.items()}


def main():
    rep, rest = sys.argv[1], sys.argv[2:]
    lcsv = rest[0] if len(rest) == 2 else None
    base = rest[-1]
    per = raw(rep)
    summ = {}
    for k, runs in per.items():
        avg = {lab: sum(r.get(lab, 0.0) for r in runs) / len(runs) for lab in KEYS.values()}
        avg["captures"] = len(runs)
        avg["dram_bytes_per_launch"] = avg["dram_read_B"] + avg["dram_write_B"]
        summ[k] = avg
    res = {"source": rep, "kernels": summ}
    if lcsv:
        res["launch_list"] = launches(lcsv)
        tot = sum(v["launches"] * v["mean_us"] for v in res["launch_list"].values())
        for v in res["launch_list"].values():
            v["share_pct"] = 100.0 * v["launches"] * v["mean_us"] / tot
    json.dump(res, open(base + ".json", "w"), indent=1)
    lines = [f"# ncu summary `{rep}`", "", "| kernel | us | DRAM B/launch | DRAM % | L1 hit % | L2 hit % | fp64 % | fma % | alu % | xu % | tensor % | occ % | regs | IPC |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, a in summ.items():
        lines.append(f"| {k} | {a['duration_ns']/1e3:.1f} | {a['dram_bytes_per_launch']:.3g} | {a['dram_pct']:.2f} | "
                     f"{a['l1_hit_pct']:.1f} | {a['l2_hit_pct']:.1f} | {a['fp64_pipe_pct']:.1f} | {a['fma_pipe_pct']:.1f} | "
                     f"{a['alu_pipe_pct']:.1f} | {a['xu_pipe_pct']:.1f} | {a['tensor_pipe_pct']:.1f} | "
                     f"{a['achieved_occupancy_pct']:.1f} | {a['registers']:.0f} | {a['ipc']:.2f} |")
    if lcsv:
        lines += ["", "Launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised):", "",
                  "| kernel | launches | mean us | share % |", "|---|---|---|---|"]
        for k, v in sorted(res["launch_list"].items(), key=lambda kv: -kv[1]["share_pct"]):
            lines.append(f"| {k[:70]} | {v['launches']} | {v['mean_us']:.1f} | {v['share_pct']:.1f} |")
    open(base + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
