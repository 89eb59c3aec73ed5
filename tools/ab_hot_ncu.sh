#!/bin/bash
# A/B of prebuilt library variants by ncu's kernel duration (high resolution;
# CUDA events on this system move in ~2 us steps): 6 launches of the C2 pass
# per variant, cold L2 per launch (ncu's default cache control).
#   bash tools/ab_hot_ncu.sh CONFIG a.so b.so ...
cfg=$1; shift
for f in "$@"; do
  FASTMAP_B200_LIB=$f ncu --metrics gpu__time_duration.sum --clock-control none -k regex:point_pass_hot \
    -c 14 --csv env FM_PASSES=14 python tools/one_pass.py full fp32 "$cfg" 2>/dev/null | grep point_pass_hot | \
    awk -F'","' -v n="$(basename "$f")" '{gsub(/"/,"",$NF); s=s" "$NF} END {print n": "s}'
done
