"""Per-kernel stall breakdown + hottest SASS lines from an ncu report (--set full, -lineinfo)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for b in blocks:
    name = next(csv.reader([b[0]]))[1]
    if kfilter and kfilter not in name:
        continue
    rows = list(csv.reader(b[1:]))
    hdr = rows[0]
    idx = {k: i for i, k in enumerate(hdr)}
    data = rows[1:]

    def f(r, k):
        try:
            return float(r[idx[k]])
        except Exception:
            return 0.0
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
    stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
    agg = sorted(((sum(f(r, k) for r in data), k) for k in stalls), reverse=True)[:6]
    print("==", name[:100])
    print("   ", ", ".join(f"{k[6:]} {v / tot * 100:.0f}%" for v, k in agg))
    top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:ntop]
    for r in top:
        s = f(r, "Warp Stall Sampling (All Samples)")
        m = sorted(((f(r, k), k) for k in stalls), reverse=True)[0]
        print(f"   {s / tot * 100:5.1f}% ex={f(r, 'Instructions Executed'):9.0f} {r[idx['Source']][:56]:56s} {m[1][6:]}")
