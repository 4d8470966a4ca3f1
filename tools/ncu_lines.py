"""Aggregate ncu warp-stall samples of one kernel by CUDA source line.

    python tools/ncu_lines.py REPORT.ncu-rep OBJ.o KERNEL_SUBSTRING [top] [MANGLED_SUBSTRING]

Maps SASS addresses in the report's source page to file:line through
`nvdisasm -g` of the object's cubin (compile with -lineinfo)."""
import csv, io, os, re, subprocess, sys, tempfile, collections

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
mangled = sys.argv[5] if len(sys.argv) > 5 else kname  # substring of the mangled name (template instance)
column = sys.argv[6] if len(sys.argv) > 6 else "Warp Stall Sampling (All Samples)"  # or e.g. stall_wait
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kname}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
ai, ci = h.index("Address"), h.index(column)
samples = []
for r in rows[hi + 1:]:
    if len(r) > ci and r[ai].startswith("0x"):
        samples.append((int(r[ai], 16), int(r[ci] or 0)))
base = min(a for a, _ in samples)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
line_of = {}
cur_fn = None
cur_line = None
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
    if m:
        cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_fn and mangled in cur_fn:
        line_of[int(m.group(1), 16)] = cur_line
agg = collections.Counter()
for a, v in samples:
    agg[line_of.get(a - base, "?")] += v
tot = sum(agg.values())
print(f"total samples {tot}")
src = {}
for k, v in agg.most_common(top):
    f, _, n = k.partition(":")
    text = ""
    if f == os.path.basename(obj).replace(".o", ".cu"):
        p = os.path.join(os.path.dirname(obj), f)
        if p not in src:
            src[p] = open(p).read().splitlines()
        text = src[p][int(n) - 1].strip()[:90] if n.isdigit() else ""
    print(f"{100 * v / tot:5.1f}%  {k:28s} {text}")
