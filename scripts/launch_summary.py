"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
per-kernel totals for the LAST step of run_step.py (launches from the last
transform launch on), in ms."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
ids = hdr.index("ID")
data = [(int(r[ids]), r[ki], float(r[vi].replace(",", ""))) for r in rows[1:] if r[vi]]
unit = rows[1][hdr.index("Metric Unit")] if len(rows) > 1 else ""
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
# the last step starts at the last transform launch (dct / gemm kernel)
dcts = [i for i, (_, k, _) in enumerate(data) if "dct" in k.split("(")[0] and "tables" not in k]
# (a DCT step also launches small gemm_f64 products for the pruning's sharper
# bound: its step starts at the DCT, a dense-transform step at its gemm)
starts = dcts or [i for i, (_, k, _) in enumerate(data) if "gemm_f64" in k]
half = data[starts[-1]:] if starts and len(sys.argv) < 3 else data
tot = collections.OrderedDict()
for _, k, v in half:
    name = k.split("(")[0].split("::")[-1][:60]
    tot[name] = tot.get(name, 0.0) + v * scale
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:9.3f} ms  {k}")
print(f"{sum(tot.values()):9.3f} ms  total ({len(half)} launches)")
