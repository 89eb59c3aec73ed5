"""Per-instruction stall samples of the hottest kernel in an ncu report.
    python tools/ncu_stalls.py rep.ncu-rep [N]   -> top-N instructions + loop listing"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
reasons = ["stall_wait", "stall_dispatch", "stall_math", "stall_short_sb", "stall_long_sb",
           "stall_not_selected", "stall_selected", "stall_branch_resolving", "stall_mio", "stall_lg"]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot = sum(int(r[col["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(f"total samples {tot}")
for r in data:
    s = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    ex = int(r[col["Instructions Executed"]] or 0)
    if ex < 1000:
        continue
    parts = " ".join(f"{k[6:]}={r[col[k]]}" for k in reasons if int(r[col[k]] or 0) > 0.15 * max(s, 1))
    print(f"{r[col['Address']][-5:]} {s:6d} {r[col['Source']].strip()[:60]:60s} {parts}")
