"""Per-SASS-instruction counters of one kernel launch from an ncu report (--set full with
source counters): instructions executed by opcode, and the hottest basic blocks (runs of
instructions between branch targets) with their share. For finding where a kernel's
warp-instructions go.  python tools/ncu_sass_hot.py REP KERNEL_REGEX [LAUNCH_SKIP] [TOP]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern,
                      "--launch-skip", str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
name = lines[0]
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ci = hdr.index("Instructions Executed")
cs = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
ins, seen = [], set()
for r in rows[1:]:
    if r and r[0] in seen:
        continue
    if r:
        seen.add(r[0])
    if len(r) <= ci:
        continue
    try:
        n = int(r[ci])
        st = int(r[cs] or 0)
    except ValueError:
        continue
    ins.append((r[0], r[src].strip(), n, st))
tot = sum(n for _, _, n, _ in ins)
stall = sum(s for *_, s in ins)
print(name[:200])
print(f"warp instructions executed: {tot/1e6:.2f} M, stall samples {stall}")
op = collections.Counter()
for _, s, n, _ in ins:
    o = s.split()[0] if not s.startswith("@") else s.split()[1]
    op[o.split(".")[0]] += n
print("by opcode:", ", ".join(f"{k} {v/tot*100:.1f}%" for k, v in op.most_common(18)))
# basic blocks: split after branches / at consecutive-count changes
blocks, cur = [], []
for a, s, n, st in ins:
    if cur and (n != cur[-1][2]):
        blocks.append(cur)
        cur = []
    cur.append((a, s, n, st))
if cur:
    blocks.append(cur)
blocks.sort(key=lambda b: -sum(x[2] for x in b))
for b in blocks[:top]:
    bt = sum(x[2] for x in b)
    bs = sum(x[3] for x in b)
    print(f"--- {bt/tot*100:5.1f}% inst, {bs/max(stall,1)*100:5.1f}% stalls, {len(b)} instr x {b[0][2]} at {b[0][0]}")
    for a, s, n, st in b[:int(sys.argv[5]) if len(sys.argv) > 5 else 12]:
        print(f"      {s[:90]:90s} {st}")
