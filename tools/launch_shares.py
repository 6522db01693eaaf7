"""Compact an ncu --metrics gpu__time_duration.sum --csv launch log into profiles/:
    python tools/launch_shares.py gpurun_out/X_launches.csv profiles/X_launches.csv profiles/X_launch_shares.txt
(id,kernel,duration_ns per launch, and per-kernel totals/shares)."""
import csv
import collections
import sys

src, out_csv, out_txt = sys.argv[1:4]
what = sys.argv[4] if len(sys.argv) > 4 else "python bench.py --steps 2 --warmup 3 --no-cpu-baseline (c2)"
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ik, iv, iid, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID"), h.index("Metric Name")
launches = []
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0].replace("void ", "").split("::")[-1]
    launches.append((int(r[iid]), name, float(r[iv].replace(",", ""))))
unit_ns = 1.0  # ncu reports ns for gpu__time_duration.sum in --csv
with open(out_csv, "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none: {what}, every launch\n")
    f.write("id,kernel,duration_ns\n")
    for i, n, v in launches:
        f.write(f"{i},{n},{v * unit_ns:.0f}\n")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for _, n, v in launches:
    tot[n] += v
    cnt[n] += 1
s = sum(tot.values())
with open(out_txt, "w") as f:
    f.write(f"per-kernel totals of {out_csv} ({what}; cold-cache serialised ncu times)\n")
    f.write(f"{'kernel':40s} {'launches':>9s} {'total ms':>10s} {'share':>7s}\n")
    for n, v in sorted(tot.items(), key=lambda x: -x[1]):
        f.write(f"{n[:40]:40s} {cnt[n]:9d} {v / 1e6:10.2f} {100 * v / s:6.1f}%\n")
print(open(out_txt).read())
