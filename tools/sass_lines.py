"""Instruction count per source line inside a kernel's main loop (needs a
-lineinfo cubin). Usage: python tools/sass_lines.py file.cubin kernel_substring [loop_rank]"""
import collections
import re
import subprocess
import sys

cub, pat = sys.argv[1], sys.argv[2]
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
# split into functions
funcs = re.split(r"\n//-+ \.text\.", out)
body = next(f for f in funcs if pat in f.split("\n", 1)[0])
ins = []
cur = "?"
labels = {}
pending = []
for line in body.split("\n"):
    lm = re.match(r"^(\.L_x_\d+):", line)
    if lm:
        pending.append(lm.group(1))
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        a = int(m.group(1), 16)
        for lab in pending:
            labels[lab] = a
        pending = []
        ins.append((a, m.group(2).strip(), cur))
loops = []
for addr, txt, _ in ins:
    m2 = re.search(r"BRA\S* (?:\S+ )?`\((\.L_x_\d+)\)", txt)
    if m2 and m2.group(1) in labels:
        tgt = labels[m2.group(1)]
        if tgt < addr:
            loops.append((tgt, addr))
loops = sorted(set(loops), key=lambda x: x[0] - x[1])
for i, (a, b) in enumerate(loops[:int(sys.argv[5]) if len(sys.argv) > 5 else 8]):
    body_i = [x[1] for x in ins if a <= x[0] <= b]
    print(f"loop {i}: {hex(a)}..{hex(b)} n={len(body_i)} DFMA={sum('DFMA' in t for t in body_i)}"
          f" BAR={sum('BAR.SYNC' in t for t in body_i)} UTMALDG={sum('UTMALDG' in t for t in body_i)}")
lo, hi = loops[rank]
cnt = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for a, t, src in ins:
    if lo <= a <= hi:
        cnt[src] += 1
        o = t.split()
        op = (o[1] if o[0].startswith("@") else o[0]).split(".")[0]
        ops[src][op] += 1
for src, n in cnt.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 40):
    print(f"{n:4d} {src:28s} " + " ".join(f"{k}:{v}" for k, v in ops[src].most_common(6)))
