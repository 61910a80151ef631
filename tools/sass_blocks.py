"""Tuning: group an ncu source page (--page source --csv --print-source sass) into
straight-line blocks and print each block's share of executed instructions and
of warp-stall samples.  Usage: python tools/sass_blocks.py page.csv [min_share%]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
lim = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h, data = rows[hi], [r for r in rows[hi + 1:] if len(r) > 5]
ia, isrc = h.index("Address"), h.index("Source")
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
num = lambda x: float(x or 0)
tot = sum(num(r[iex]) for r in data)
tots = sum(num(r[iss]) for r in data) or 1
print(f"executed {tot:.3e} warp-instructions, {tots:.0f} stall samples")
blocks = []
for r in data:
    ex, st = num(r[iex]), num(r[iss])
    if blocks and abs(blocks[-1][1] - ex) <= 0.02 * max(ex, 1):
        blocks[-1][2] += 1
        blocks[-1][3] += st
        blocks[-1][5] = r[isrc]
    else:
        blocks.append([r[ia], ex, 1, st, r[isrc], r[isrc]])
for b in blocks:
    share = b[1] * b[2] / tot * 100
    if share > lim or b[3] / tots * 100 > 2 * lim:
        print(f"{b[0][-5:]} n={b[2]:3d} x{b[1] / 1e6:7.2f}M inst={share:5.1f}% stall={b[3] / tots * 100:5.1f}%  "
              f"{b[4].strip()[:44]} .. {b[5].strip()[:36]}")
