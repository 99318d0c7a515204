"""Summarise an ncu report: key metrics, stall reasons, and the SASS opcode histogram."""
import collections, csv, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, vals = rows[0], rows[2] if len(rows) > 2 else rows[1]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum"]
out = {}
for i, h in enumerate(hdr):
    if h in want:
        out[h] = vals[i]
for k in want:
    if k in out:
        print(f"{k:70s} {out[k]}")
st = {h: vals[i] for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
tot = sum(float(v or 0) for v in st.values())
print("stall samples (share):")
for h, v in sorted(st.items(), key=lambda x: -float(x[1] or 0))[:10]:
    print(f"   {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {float(v)/tot*100:5.1f}%")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]; data = rows[2:]
ie = hdr.index("Instructions Executed"); sc = hdr.index("Source")
c = collections.Counter(); tot = 0
for r in data:
    try: n = int(r[ie])
    except: continue
    t = r[sc].replace(',', ' ').split()
    if not t: continue
    o = t[1] if t[0].startswith('@') else t[0]
    c[o] += n; tot += n
print("instructions executed:", tot)
for o, n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"   {o:28s} {n:12d} {n/tot*100:5.1f}%")
