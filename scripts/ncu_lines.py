"""Aggregate ncu per-SASS metrics (page source --print-source sass) onto CUDA
source lines using the mixed cuda,sass view.  Usage:
  python scripts/ncu_lines.py REPORT.ncu-rep [kernel-substring]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
def run(src):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", src],
                         capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))
mix = run("cuda,sass")
addr2line, line_src, cur = {}, {}, None
for r in mix:
    if len(r) >= 4 and r[0] and r[0].isdigit():
        cur = int(r[0]); line_src[cur] = r[1]
    elif len(r) >= 4 and r[2].startswith("0x"):
        addr2line[r[2]] = cur
sass = run("sass")
hdr = None
agg = collections.defaultdict(lambda: [0, 0, 0])
for r in sass:
    if r and r[0] == "Address":
        hdr = r; continue
    if hdr is None or not r or not r[0].startswith("0x"):
        continue
    d = dict(zip(hdr, r))
    ln = addr2line.get(r[0])
    def num(k):
        try: return float(d.get(k, "0") or 0)
        except ValueError: return 0.0
    agg[ln][0] += num("Instructions Executed")
    agg[ln][1] += num("Warp Stall Sampling (All Samples)")
    agg[ln][2] += num("L1 Wavefronts Shared Excessive")
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"{'line':>5} {'inst%':>6} {'stall%':>6} {'shexc':>10}  source")
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][int(sys.argv[3]) if len(sys.argv) > 3 else 1])[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{str(ln):>5} {100*v[0]/tot_i:6.2f} {100*v[1]/tot_s:6.2f} {v[2]:10.0f}  {line_src.get(ln, '')[:90]}")
