"""Summarise one ncu --set full capture of the tile kernel for profiles/:
time, DRAM traffic, achieved bandwidth, issue/occupancy, stall mix, pipes.
    python scripts/ncu_summary.py REPORT.ncu-rep OUT.md [alg_bytes_per_launch]"""
import csv, json, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
def f(k):
    try: return float(d[k])
    except (KeyError, ValueError): return None
t_ms = f("gpu__time_duration.sum")
t_unit = u.get("gpu__time_duration.sum", "")
t_s = t_ms * {"msecond": 1e-3, "ms": 1e-3, "usecond": 1e-6, "us": 1e-6, "s": 1.0, "second": 1.0}.get(t_unit, 1e-9)
rd = f("dram__bytes_read.sum"); wr = f("dram__bytes_write.sum")
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}
rd_b = rd * scale.get(u.get("dram__bytes_read.sum"), 1); wr_b = wr * scale.get(u.get("dram__bytes_write.sum"), 1)
stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v or 0) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(stalls.values()) or 1
lines = [f"# ncu --set full: `{d.get('Kernel Name', '?')[:80]}`", "",
         f"report: `{rep.split('/')[-1]}` (cold-cache replay; `--clock-control none`)", "",
         "| metric | value |", "|---|---|",
         f"| duration | {t_s*1e3:.3f} ms |",
         f"| DRAM read / write | {rd_b/1e9:.3f} / {wr_b/1e9:.3f} GB |",
         f"| DRAM bandwidth (traffic / duration) | {(rd_b+wr_b)/t_s/1e9:.0f} GB/s |"]
if alg:
    lines.append(f"| algorithmic bytes / launch | {alg/1e9:.3f} GB ({alg/t_s/1e9:.0f} GB/s) |")
for k, name in [("launch__registers_per_thread", "registers / thread"), ("launch__block_size", "block"),
                ("launch__grid_size", "grid"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
                ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
                ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / cycle / SMSP"),
                ("smsp__inst_executed.sum", "warp instructions"),
                ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
                ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
                ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
                ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu pipe %")]:
    if k in d: lines.append(f"| {name} | {d[k]} |")
lines += ["", "stall mix (pc sampling):", "", "| reason | share |", "|---|---|"]
for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]:
    lines.append(f"| {k} | {100*v/tot:.1f}% |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
print(json.dumps({"dram_bytes_per_launch": rd_b + wr_b}))
