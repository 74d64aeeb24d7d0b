"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch).

Prints (1) one step's launches -- the last window between two image-layer forward launches (each
training step starts with exactly one) that contains the head -- grouped by kernel with its share of that step, then
(2) the full per-launch list.  ncu serialises launches and runs them cold, so the shares, not the
absolute times, are what compare with the live bench timing.
"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            out.append((d['Kernel Name'][:70], float(d['Metric Value'].replace(',', ''))))

# a training step starts with the image layer's forward (conv1_fwd_kernel; im2col_kernel in other modes).
# bench.py's later legs replay the step without the FC / softmax head (the conv-stage breakdown) and
# single passes, so the window taken is the last one that holds a head kernel: a whole training step.
starts = [i for i, (n, _) in enumerate(out) if 'im2col_kernel' in n or 'conv1_fwd_kernel' in n]
HEAD = ('fc_fwd_partial', 'softmax_xent', 'oneshot_allreduce')
def _end(a, b):   # a step ends with its SGD launch (if the window runs on into other legs)
    for i in range(a, b):
        if 'sgd_multi' in out[i][0]:
            return i + 1
    return b
wins = [(a, _end(a, b)) for a, b in zip(starts, starts[1:] + [len(out)])
        if any(h in n for n, _ in out[a:b] for h in HEAD)]
if wins or len(starts) >= 2:
    a, b = wins[-1] if wins else (starts[-2], starts[-1])
    step = out[a:b]
    tot = sum(v for _, v in step)
    agg = OrderedDict()
    for n, v in step:
        c, t = agg.get(n, (0, 0.0))
        agg[n] = (c + 1, t + v)
    print(f"one step (launches {a}..{b - 1}): {len(step)} launches, {tot / 1e3:.1f} us serialised")
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {t / 1e3:9.1f} us {100 * t / tot:5.1f}%  x{c:<3d} {n}")
    print()

tot = sum(v for _, v in out)
print(f"all: {len(out)} launches, total {tot / 1e3:.1f} us")
for n, v in out:
    print(f"{v / 1e3:9.1f} us {100 * v / tot:5.1f}%  {n}")
