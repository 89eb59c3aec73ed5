#!/bin/bash
# A/B the fused pass across prebuilt library variants, interleaved rounds:
#   bash tools/ab_hot.sh CONFIG ROUNDS build_variants/a.so build_variants/b.so ...
cfg=$1; rounds=$2; shift 2
for r in $(seq "$rounds"); do
  for f in "$@"; do
    printf "%s %s " "$r" "$(basename "$f")"
    FASTMAP_B200_LIB=$f python tools/pass_probe.py "$cfg" - 2>&1 | tail -1
  done
done
