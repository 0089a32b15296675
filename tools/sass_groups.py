import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
blocks = []; cur = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r]; blocks.append(cur)
    elif cur is not None:
        cur.append(r)
b = blocks[which]
print(b[0][1][:100])
h = b[1]; data = [r for r in b[2:] if len(r) > 10]
ie = h.index("Instructions Executed"); src = h.index("Source"); ws = h.index("Warp Stall Sampling (All Samples)")
f = lambda x: float(x.replace(',', '') or 0)
tot = sum(f(r[ie]) for r in data); tots = sum(f(r[ws]) for r in data)
print("total", tot, len(data), "stall samples", tots)
grp = []
for i, r in enumerate(data):
    c = f(r[ie])
    if grp and grp[-1][1] == c: grp[-1][2] += 1; grp[-1][4] += f(r[ws])
    else: grp.append([i, c, 1, r[src][:50], f(r[ws])])
for g in grp:
    if g[1] * g[2] > tot * 0.01 or g[4] > tots * 0.03:
        print(f"start {g[0]:5d} count {g[1]:9.0f} n {g[2]:4d} share {100*g[1]*g[2]/tot:5.1f}% stall {100*g[4]/max(tots,1):5.1f}%  {g[3]}")
if len(sys.argv) > 4:
    for r in data[int(sys.argv[3]):int(sys.argv[4])]: print(r[ie], r[src][:90])
