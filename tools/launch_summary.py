import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
h = rows[hi]; data = rows[hi + 1:]
ki = h.index('Kernel Name'); vi = h.index('Metric Value')
seq = [(r[ki][:48], float(r[vi].replace(',', '')) / 1e3) for r in data if len(r) > vi]
nf = 0; start = 0
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 8
for i, (k, v) in enumerate(seq):
    if 'forward_kernel' in k:
        nf += 1
        if nf == skip + 1: start = i; break
while start > 0 and 'forward_kernel' not in seq[start][0]: start -= 1
# back up to the cull of that iteration
j = start
while j > 0 and 'cull_kernel' not in seq[j][0]: j -= 1
agg = defaultdict(lambda: [0, 0.0])
for k, v in seq[j:]:
    agg[k][0] += 1; agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v:9.1f}us {c:3d} {100*v/tot:5.1f}%  {k}")
print("total us", round(tot, 1))
