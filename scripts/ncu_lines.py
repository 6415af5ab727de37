"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: python scripts/ncu_lines.py REPORT.ncu-rep CUBIN KERNEL_SUBSTRING [top]
The SASS rows of `ncu --page source --print-source sass` are in address order;
nvdisasm -g gives the source line of each instruction of the same cubin."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
fname = sys.argv[5] if len(sys.argv) > 5 else kname  # substring of the mangled name in the cubin
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
# several kernels: take the first SASS section whose "Kernel Name" line matches
start = next(i for i, x in enumerate(r) if x and x[0] == "Kernel Name" and kname in x[1]) + 1
end = next((i for i in range(start + 1, len(r)) if r[i] and r[i][0] == "Kernel Name"), len(r))
hdr, rows = r[start], r[start + 1:end]
si = hdr.index("Warp Stall Sampling (All Samples)")
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# find the function section
lines = dis.splitlines()
fun = None
cur_line = None
seq = []
for ln in lines:
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        fun = m.group(1)
        continue
    if fun is None or fname not in fun:
        continue
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
    if m:
        cur_line = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
        seq.append(cur_line)
print("ncu rows", len(rows), "sass instrs", len(seq))
tot = sum(float(x[si] or 0) for x in rows)
reasons = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.Counter()
why = collections.defaultdict(collections.Counter)
for k, x in enumerate(rows):
    if k < len(seq):
        agg[seq[k]] += float(x[si] or 0)
        for c in reasons:
            why[seq[k]][hdr[c][6:]] += float(x[c] or 0)
for key, v in agg.most_common(top):
    w = ", ".join(f"{n} {100 * c / max(v, 1):.0f}%" for n, c in why[key].most_common(3) if c > 0)
    print(f"{100 * v / tot:5.1f}%  {key:32s} {w}")
