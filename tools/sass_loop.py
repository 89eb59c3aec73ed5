"""Opcode histogram of the main loop (largest backward-branch body) of a kernel.
    python tools/sass_loop.py <cubin|so|o> <kernel-name-substring>"""
import collections, re, subprocess, sys
sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout.split("\n")
st = [i for i, l in enumerate(sass) if "Function :" in l and sys.argv[2] in l][0]
en = next((i for i, l in enumerate(sass[st + 1:], st + 1) if "Function :" in l), len(sass))
ins = []
for l in sass[st:en]:
    m = re.match(r"\s+/\*([0-9a-f]{4})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
best = None
for a, t in ins:
    m = re.search(r"BRA(?:\.U)? (?:!?U?P\d, )?(0x[0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        lo = int(m.group(1), 16)
        if best is None or a - lo > best[1] - best[0]:
            best = (lo, a)
body = [t for a, t in ins if best[0] <= a <= best[1]]
c = collections.Counter()
for t in body:
    w = t.split()
    op = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
    c[op] += 1
print(f"loop {best[0]:#x}-{best[1]:#x}: {len(body)} instructions")
print(", ".join(f"{k} {v}" for k, v in c.most_common()))
if len(sys.argv) > 3:
    print("\n".join(body))
