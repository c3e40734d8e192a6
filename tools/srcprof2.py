"""Per-source-line instruction / stall shares of an ncu report (needs -lineinfo
and --import-source on):  python tools/srcprof2.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True).stdout.decode(errors="replace")
fn = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr and r and r[0].isdigit():
        try:
            k = (fn, int(r[0]))
            agg[k][0] += int(r[ii] or 0)
            agg[k][1] += int(r[si] or 0)
            agg[k][2] = r[1][:100]
        except (ValueError, IndexError):
            pass
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print("warp instructions", tot, "stall samples", ts)
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}%i {v[1] / ts * 100:5.1f}%s {k[0]}:{k[1]} {v[2]}")
