"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; out = []
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            out.append((d['Kernel Name'][:70], float(d['Metric Value'].replace(',', ''))))
tot = sum(v for _, v in out)
print(f"{len(out)} launches, total {tot/1e3:.1f} us")
for n, v in out: print(f"{v/1e3:9.1f} us {100*v/tot:5.1f}%  {n}")
