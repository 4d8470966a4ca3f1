"""Print the kernels of the last frame in an ncu gpu__time_duration launch list."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
H = rows[h]; ki = H.index('Kernel Name'); vi = H.index('Metric Value'); mi = H.index('Metric Name')
seq = [(r[ki], float(r[vi].replace(',', ''))) for r in rows[h + 1:] if len(r) > vi and r[mi] == 'gpu__time_duration.sum']
idx = [i for i, (k, v) in enumerate(seq) if 'k_camera_rays' in k]
tot = 0.0
for k, v in seq[idx[-1]:]:
    tot += v
    print(f"{v / 1000:8.1f} us  {k[:70]}")
print(f"sum {tot / 1000:.1f} us")
