"""Turns the JSON lines that tests/gpu_util.check_frame appends to $GS_PARITY_LOG into the
parity table (markdown): per frame checked, the all-pixel max |d|, the count of pixels
above 2e-3 (each flagged and within its flip bound), the flagged fraction, the max |d| on
unflagged pixels and the PSNR.  python tools/parity_table.py LOG > OUT.md"""
import json
import sys

rows = [json.loads(line) for line in open(sys.argv[1])]
print("| frame | pixels | max abs (all) | px > 2e-3 | of which unflagged | flagged % | max abs (unflagged) "
      "| max abs T (unflagged) | PSNR dB |")
print("|---|---|---|---|---|---|---|---|---|")
for r in sorted(rows, key=lambda r: r["case"]):
    print(f"| {r['case']} | {r['n_pixels']} | {r['max_all']:.2e} | {r['n_over']} | {r['over_unflagged']} | "
          f"{100 * r['flagged']:.3f} | {r['max_unflagged']:.2e} | {r['T_max']:.2e} | {r['psnr']:.1f} |")
w = max(rows, key=lambda r: r["max_all"])
f = max(rows, key=lambda r: r["flagged"])
print(f"\n{len(rows)} frames; worst all-pixel max abs {w['max_all']:.2e} ({w['case']}); "
      f"pixels above 2e-3 in total {sum(r['n_over'] for r in rows)} (unflagged: {sum(r['over_unflagged'] for r in rows)}); "
      f"largest flagged fraction {100 * f['flagged']:.3f} % ({f['case']}); min PSNR {min(r['psnr'] for r in rows):.1f} dB")
