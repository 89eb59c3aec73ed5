#!/bin/bash
# Interleaved A/B of prebuilt library variants with batched timing:
#   bash tools/ab_hot_batch.sh CONFIG ROUNDS a.so b.so ...
cfg=$1; rounds=$2; shift 2
for r in $(seq "$rounds"); do
  for f in "$@"; do
    printf "%s %s " "$r" "$(basename "$f")"
    FASTMAP_B200_LIB=$f python tools/pass_probe_batch.py "$cfg" 20 10 2>&1 | tail -1
  done
done
