"""Summarise an ncu report (--set full) and a launch list into markdown for
profiles/.  Runs here (no GPU): ncu -i <rep> --page raw/source --csv.

    python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep [gpurun_out/launches_X.csv] > profiles/X.md
"""

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe % (active)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % (active)"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % (active)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe % (active)"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % (active)"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__cycles_active.avg", "SMSP active cycles"),
    ("sm__cycles_elapsed.avg", "SM elapsed cycles"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = ncu_csv(["-i", rep, "--page", "raw"])
    head, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(head, vals))
    u = dict(zip(head, units))
    print(f"## ncu --set full: `{d.get('Kernel Name', '?')[:120]}`\n")
    print("| metric | value |\n|---|---|")
    for k, name in KEYS:
        if k in d:
            print(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
    stalls = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v))
              for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("not_issued") and v.replace(".", "").isdigit()]
    stalls.sort(key=lambda x: -x[1])
    tot = sum(v for _, v in stalls) or 1.0
    print("\nTop warp stall reasons (pc sampling):\n")
    for k, v in stalls[:8]:
        print(f"- {k}: {100 * v / tot:.1f}%")
    src = ncu_csv(["-i", rep, "--page", "source", "--print-source", "sass"])
    if len(src) > 2:
        h = src[1]
        ix, isrc = h.index("Instructions Executed"), h.index("Source")
        ops = collections.Counter()
        for r in src[2:]:
            # multi-kernel reports repeat the header row per kernel: skip it
            if len(r) > ix and r[isrc].split() and (r[ix] or "0").isdigit():
                t = r[isrc].split()
                op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
                ops[op] += int(r[ix] or 0)
        total = sum(ops.values())
        print(f"\nSASS opcode mix ({total} warp instructions):\n")
        print(", ".join(f"{op} {100 * n / total:.1f}%" for op, n in ops.most_common(14)))
        proof = [op for op in ("UBLKCP", "SYNCS", "UTMALDG", "LDGSTS", "DFMA", "FFMA2", "FADD2", "FMUL2", "HMMA", "UTCHMMA") if ops.get(op)]
        print(f"\nBlackwell evidence in SASS: {', '.join(proof)}")
    if len(sys.argv) > 2:
        rows = list(csv.reader(open(sys.argv[2])))
        try:
            h = next(r for r in rows if "Kernel Name" in r)
            ik, iv = h.index("Kernel Name"), h.index("Metric Value")
            agg = collections.defaultdict(list)
            for r in rows[rows.index(h) + 1:]:
                if len(r) > iv:
                    agg[r[ik].split("(")[0][:70]].append(float(r[iv].replace(",", "")))
            tot = sum(sum(v) for v in agg.values())
            print("\nLaunch list (ncu --metrics gpu__time_duration.sum, cold/serialised):\n")
            print("| kernel | launches | total ns | share |\n|---|---|---|---|")
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:12]:
                print(f"| `{k}` | {len(v)} | {sum(v):.0f} | {100 * sum(v) / tot:.1f}% |")
        except StopIteration:
            pass


if __name__ == "__main__":
    main()
