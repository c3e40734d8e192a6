"""Top SASS instructions of an ncu report by one stall reason (or all samples).

    python tools/stallsass.py report.ncu-rep [column, default 'Warp Stall Sampling (All Samples)'] [top]
Columns: e.g. stall_long_sb, stall_wait, stall_barrier, stall_short_sb, Instructions Executed.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "Warp Stall Sampling (All Samples)"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True).stdout.decode(errors="replace")
rows, hdr = [], None
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] in ("Address", "# Address"):
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        rows.append(dict(zip(hdr, r)))
if not rows:
    sys.exit("no SASS rows")
tot = sum(float(x.get(col) or 0) for x in rows)
rows.sort(key=lambda x: -float(x.get(col) or 0))
print(f"{col}: total {tot:.0f}")
for x in rows[:top]:
    v = float(x.get(col) or 0)
    print(f"{100 * v / max(tot, 1):5.1f}%  {x.get('Address', ''):>8}  {x.get('Source', '')[:110]}")
