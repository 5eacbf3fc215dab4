"""List the CALL sites (division slow paths, subroutines) a kernel executed, with counts.

usage: python tools/slowpath_calls.py REPORT.ncu-rep OBJ.o MANGLED_KERNEL_SUBSTR
Needs the object file of the profiled build (-lineinfo)."""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kern = sys.argv[1:4]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, data = rows[1], rows[2:]
ia, ie, isrc = h.index("Address"), h.index("Instructions Executed"), h.index("Source")
base = int(data[0][ia], 16)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = glob.glob(os.path.join(d, "*.cubin"))[0]
lines = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout.splitlines()
st = [i for i, l in enumerate(lines) if ".section" in l and ".text." in l and kern in l][0]
en = next((i for i, l in enumerate(lines) if i > st + 5 and ".section" in l and ".text." in l), len(lines))
cur, off2line, fn, curfn = None, {}, {}, "main"
for l in lines[st:en]:
    m = re.search(r'//## File ".*/(\S+)", line (\d+)', l)
    if m:
        cur = m.group(1) + ":" + m.group(2)
    if ".type" in l and "@function" in l:
        curfn = l.split()[1]
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
        fn[int(m.group(1), 16)] = curfn
tot, per_fn = 0, {}
for r in data:
    off, n = int(r[ia], 16) - base, int(r[ie])
    tot += n
    per_fn[fn.get(off, "?")] = per_fn.get(fn.get(off, "?"), 0) + n
    if "CALL" in r[isrc] and n > 0:
        print(f"{off:#7x} {off2line.get(off)!s:28s} {n:12d}  {r[isrc].strip()[:60]}")
for k, v in per_fn.items():
    print(f"{100.0 * v / max(tot, 1):5.1f}%  {k[:90]}")
