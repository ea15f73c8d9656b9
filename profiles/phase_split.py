"""Per-phase instruction / stall-sample split of an ncu report of fast128_kernel.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
       python profiles/phase_split.py src.csv ITEMS [KERNEL_SOURCE_PATH]
SASS instructions are sorted by address and assigned to the phase of the
nearest preceding holo_fast.cu source line (inlined FFT helpers inherit it).
"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
items = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
src_path = sys.argv[3] if len(sys.argv) > 3 else rows[0][1]
markers = {}
for i, line in enumerate(open(src_path), 1):
    m = re.search(r"// [-=]+ (row pass|producer|consumer|drain D|column pass|IFFT|removal phase|HG overlap)", line)
    if re.search(r"__global__ void", line) and "kernel_line" not in markers.values():
        markers[i] = "setup"
        kernel_start = i
    if m:
        markers[i] = m.group(1)
hdr = rows[2]
ii = hdr.index("Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
f = src_path.split("/")[-1]
ln = None
ins = []
for r in rows[3:]:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) < 6:
        continue
    if r[0] != "":
        try:
            ln = int(r[0])
        except ValueError:
            ln = None
        continue
    if r[2] in ("...", "-"):
        continue
    try:
        ins.append((int(r[2], 16), f, ln, int(r[ii]), int(r[si])))
    except ValueError:
        pass
# an inlined instruction is listed under every source line that claims it: keep one
# copy per address, preferring the kernel's own file
best = {}
main = src_path.split("/")[-1]
for a, fname, line, n, s in ins:
    if a not in best or (fname == main and best[a][0] != main):
        best[a] = (fname, line, n, s)
ins = sorted((a,) + v for a, v in best.items())
bounds = sorted(markers)


def phase_of(line):
    name = "setup"
    for b in bounds:
        if line >= b:
            name = markers[b]
    return name


first = min(markers)   # lines before the kernel body are inlined helpers: they inherit the phase
cur = "setup"
tot, st = {}, {}
for a, fname, line, n, s in ins:
    if fname == main and line is not None and line >= first:
        cur = phase_of(line)
    tot[cur] = tot.get(cur, 0) + n
    st[cur] = st.get(cur, 0) + s
T, S = sum(tot.values()), sum(st.values())
for k in tot:
    print(f"{k:14s} warp-inst/item {tot[k] / items:9.0f} ({100 * tot[k] / T:4.1f}%)  stall samples {100 * st[k] / S:4.1f}%")
print(f"total warp-inst/item {T / items:.0f}")
