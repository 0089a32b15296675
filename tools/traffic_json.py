"""profiles/ncu_traffic.json from an ncu launch list of tools/probe_only.py captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum: DRAM bytes per call of
each probed ABI entry point (sum over the kernels it launches; median over the second half of the
launches of each kernel, i.e. steady state)."""
import csv
import json
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) > vi:
        per[(int(r[ii]), r[ki])][r[mi]] = float(r[vi].replace(",", ""))
byk = defaultdict(list)
for (i, k), m in sorted(per.items()):
    byk[k].append((m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0),
                   m.get("gpu__time_duration.sum", 0.0)))


def med(k):
    xs = byk[k][len(byk[k]) // 2:]
    xs = sorted(xs, key=lambda t: t[0] + t[1])
    return xs[len(xs) // 2]


def find(sub):
    return [k for k in byk if sub in k]


ops = {
    "frustum_cull": ["cull_kernel"],
    "deferred_update": ["update_kernel<16, 0>", "walk4_kernel<16, 0>"],
    "restore_view": ["restore_kernel<16>"],
    "geo deferred_update (defer_max=0)": ["dense_update_kernel<16>"],
}
out = {"_source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none, python tools/probe_only.py (bench.py kernel_probe workload: 4M Gaussians, "
                  "8.28% sparse grads, steady state); median over the second half of the launches; bytes per call of "
                  "the ABI entry point (all kernels it launches, incl. the id-list index_kernel where used)"}
idx = find("index_kernel")
for op, subs in ops.items():
    ks = {}
    for s in subs:
        for k in find(s):
            r, w, t = med(k)
            ks[k.split("(")[0].replace("void ", "").replace("gssd::<unnamed>::", "")] = [r, w, t]
    if op != "frustum_cull" and idx:
        r, w, t = med(idx[0])
        ks["index_kernel"] = [r, w, t]
    out[op] = {"dram_bytes": sum(v[0] + v[1] for v in ks.values()), "kernels": ks}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
