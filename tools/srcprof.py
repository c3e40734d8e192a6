"""Summarise an `ncu --page source --csv --print-source=cuda,sass` dump by source line."""
import csv
import sys

rows = []
fn = None
with open(sys.argv[1]) as f:
    for r in csv.reader(f):
        if len(r) >= 2 and r[0] == 'File Path':
            fn = r[1].split('/')[-1]
            continue
        if len(r) < 8 or r[0] in ('Line No',) or not r[0]:
            continue
        try:
            inst = int(r[7]); samp = int(r[4])
        except ValueError:
            continue
        rows.append((inst, samp, fn, r[0], r[1][:110]))
tot = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print('total warp inst', tot, 'stall samples', ts)
key = 1 if len(sys.argv) > 2 and sys.argv[2] == 'stall' else 0
for x in sorted(rows, key=lambda x: -x[key])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{x[0]/tot*100:5.1f}%i {x[1]/ts*100:5.1f}%s {x[2]}:{x[3]} {x[4]}")
