"""Stall samples / executed instructions of an `ncu --page source --csv --print-source=sass` dump,
per region between mbarrier operations, plus the top instructions.

    python tools/sass_regions.py dump.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
ok = [r for r in data if r[iS].isdigit()]
tot = sum(int(r[iS]) for r in ok) or 1
print("samples", tot, "warp inst", sum(int(r[iE]) for r in ok))
acc = acci = 0
start = 0
for i, r in enumerate(ok):
    acc += int(r[iS])
    acci += int(r[iE])
    src = r[1].strip()
    if "SYNCS" in src or "EXIT" in src or "BAR.SYNC" in src or i == len(ok) - 1:
        if acc or acci:
            print(f"{start:5d}-{i:5d} samples {acc / tot * 100:5.1f}%  warp-inst {acci:10d}  ends with {src[:60]}")
        acc = acci = 0
        start = i + 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lst = sorted(((int(r[iS]), i, r[1].strip(), int(r[iE])) for i, r in enumerate(ok)), reverse=True)[:top]
for s_, i, src, e in lst:
    print(f"{s_ / tot * 100:5.1f}% {i:5d} {e:9d} {src[:90]}")
