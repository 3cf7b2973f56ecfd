"""One-page summary of an ncu --set full capture (first kernel in the report):
duration, DRAM traffic, pipe utilisation, occupancy and top stall reasons.
usage: python scripts/ncu_summary.py report.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, val = rows[0], rows[1], rows[2]
get = {h: (v, u) for h, v, u in zip(hdr, val, units)}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_src_fp64.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
print(" ".join(sys.argv[2:]) or rep)
print(f"kernel: {val[hdr.index('Kernel Name')]}")
for k in keys:
    if k in get:
        v, u = get[k]
        print(f"  {k:78s} {v} {u}")
stalls = sorted(((h, v) for h, v in zip(hdr, val)
                 if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")),
                key=lambda hv: -float(hv[1] or 0))[:10]
print("top stall reasons (warps per issue-active cycle):")
for h, v in stalls:
    print(f"  {h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} {float(v):.3f}")
