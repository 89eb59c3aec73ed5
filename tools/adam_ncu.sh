#!/bin/bash
# Under gpurun: warm-cache per-kernel durations of the Adam step (ncu launch
# list over tools/adam_probe.py), summarised per kernel.  Usage: adam_ncu.sh c2 [c4 ...]
mkdir -p gpurun_out
for c in "$@"; do
  timeout 400 ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --cache-control none -k regex:"pair_grad|image_reduce" -c 40 --csv \
    --log-file gpurun_out/adam_$c.csv python tools/adam_probe.py $c fp32 2 > /dev/null 2>&1
  python - "$c" <<'PY'
import csv, collections, io, sys
c = sys.argv[1]
txt = open(f"gpurun_out/adam_{c}.csv").read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
d = collections.defaultdict(list)
for r in rows:
    d[(r["Kernel Name"].split("(")[0][-28:], r["Metric Name"][:24])].append(float(r["Metric Value"].replace(",", "")))
for k, v in sorted(d.items()):
    v.sort(); print(c, k, "median", v[len(v) // 2], "n", len(v))
PY
done
