"""Group an ncu SASS source page (csv) into runs of equal execution count: where the
instructions and the stall samples of a kernel go. Usage: sass_hot.py page.csv [min_G]"""
import csv, sys
r = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
hdr = r[1]; rows = r[2:]
ia = hdr.index("Instructions Executed"); src = hdr.index("Source")
smp = hdr.index("Warp Stall Sampling (All Samples)")
groups = []
for i, x in enumerate(rows):
    c = int(x[ia])
    if groups and groups[-1][1] == c:
        g = groups[-1]; g[2] += 1; g[3].append(x[src].strip()); g[4] += int(x[smp])
    else:
        groups.append([i, c, 1, [x[src].strip()], int(x[smp])])
tot = sum(int(x[ia]) for x in rows); ts = sum(int(x[smp]) for x in rows)
print(f"total {tot/1e9:.2f}G instructions, {ts} samples")
for g in groups:
    t = g[1] * g[2]
    if t > thr * 1e9 or g[4] / ts > 0.01:
        print(f"idx {g[0]:5d} {g[1]/1e6:8.2f}M x{g[2]:3d} = {t/1e9:5.2f}G samp {g[4]/ts*100:5.1f}%  "
              f"{g[3][0][:38]} .. {g[3][-1][:38]}")
