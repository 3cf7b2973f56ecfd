"""Top SASS instructions by warp-stall samples of an ncu report (source page),
with the long-scoreboard share.  usage: ncu_source_top.py report.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
si, ns = h.index("Source"), h.index("# Samples")
keys = [k for k in ("stall_long_sb", "stall_wait", "stall_math", "stall_barrier", "stall_short_sb", "stall_lg") if k in h]
data = []
for r in rows[2:]:
    try:
        data.append((float(r[ns] or 0), r[si][:90], [float(r[h.index(k)] or 0) for k in keys]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1.0
print("total samples", tot, "keys", keys)
for i, (v, s, ks) in enumerate(data):
    data[i] = (v, s, ks, i)
for v, s, ks, i in sorted(data, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}%  #{i:5d} {s:90s} " + " ".join(f"{int(x):6d}" for x in ks))
