"""Static SASS instruction mix of a kernel's main loop (largest backward
branch span). Usage: python tools/sass_loop.py file.cubin kernel_substring"""
import collections
import re
import subprocess
import sys

cub, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
body = next(f for f in funcs if pat in f.split("\n", 1)[0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
loops = []
for addr, txt in ins:
    m = re.search(r"BRA (?:\S+ )?0x([0-9a-f]+)", txt)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < addr:
            loops.append((tgt, addr))
want = sys.argv[3] if len(sys.argv) > 3 else None
for lo, hi in sorted(loops, key=lambda x: x[0] - x[1])[:4]:
    loop = [t for a, t in ins if lo <= a <= hi]
    if want and not any(want in t for t in loop):
        continue
    cnt = collections.Counter()
    for t in loop:
        op = t.split()
        o = op[1] if op[0].startswith("@") else op[0]
        cnt[o.split(".")[0]] += 1
    dp = sum(cnt[k] for k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"))
    print(f"loop {hex(lo)}..{hex(hi)}: {len(loop)} instructions, FP64 {dp}, other {len(loop) - dp}")
    print("   " + ", ".join(f"{k} {v}" for k, v in cnt.most_common(40)))
