#!/bin/bash
# Registers / spills of the hot point-pass kernels: tools/ptxas_regs.sh [extra nvcc flags]
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include -Xptxas -v "$@" \
  -c paper_2505_04612_b200/csrc/fm_point_pass.cu -o /tmp/pp.o 2>&1 | python3 -c '
import re,sys
cur=None
for l in sys.stdin:
    m=re.search(r"Compiling entry function .(\S+).", l)
    if m: cur=m.group(1); continue
    m=re.search(r"point_pass_hotILj(\d+)ELb(\d)ELi(\d+)", cur or "")
    if not m: continue
    if "spill" in l: sp=re.search(r"(\d+) bytes spill stores", l).group(1)
    r=re.search(r"Used (\d+) registers", l)
    if r: print(f"mode {m.group(1):>3} mom64={m.group(2)} L={m.group(3):>2}: {r.group(1)} regs, spill {sp}")
'
