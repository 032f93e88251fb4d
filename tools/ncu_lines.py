"""Top source lines of one kernel in an ncu capture (needs -lineinfo)."""
import csv, subprocess, sys, io
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None; data = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            key = (cur, r[0])
            a = data.setdefault(key, [0, 0, r[1][:100]])
            a[0] += int(r[6] or 0); a[1] += int(r[7] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in data.values()) or 1; toti = sum(v[1] for v in data.values()) or 1
print("samples", tot, "warp-instr", toti)
for (f, l), (s, i, src) in sorted(data.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{s/tot*100:5.1f}% {i/toti*100:5.1f}%i {f[:14]}:{l:>4} {src}")
