"""Opcode histogram of the main loop (largest backward-branch body) of a kernel.
    python tools/sass_loop.py <cubin|so|o> <kernel-name-substring> [x | top]
x: also print the loop body; top: histograms of the 4 largest loops."""
import collections, re, subprocess, sys
sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout.split("\n")
st = [i for i, l in enumerate(sass) if "Function :" in l and sys.argv[2] in l][0]
en = next((i for i, l in enumerate(sass[st + 1:], st + 1) if "Function :" in l), len(sass))
ins = []
for l in sass[st:en]:
    m = re.match(r"\s+/\*([0-9a-f]{4})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
loops = []
for a, t in ins:
    m = re.search(r"BRA(?:\.U)? (?:!?U?P\d, )?(0x[0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        loops.append((int(m.group(1), 16), a))
loops.sort(key=lambda x: x[1] - x[0], reverse=True)
mode = sys.argv[3] if len(sys.argv) > 3 else ""
for lo, hi in loops[:4 if mode == "top" else 1]:
    body = [t for a, t in ins if lo <= a <= hi]
    c = collections.Counter()
    for t in body:
        w = t.split()
        c[(w[1] if w[0].startswith("@") else w[0]).split(".")[0]] += 1
    print(f"loop {lo:#x}-{hi:#x}: {len(body)} instructions")
    print(", ".join(f"{k} {v}" for k, v in c.most_common()))
    if mode == "x":
        print("\n".join(body))
