"""Attribute ncu per-instruction counters (source page, SASS) to CUDA source lines.

usage: python tools/sass_hotspots.py REPORT.ncu-rep OBJ.o KERNEL_SUBSTR [top]
Needs the object file of the profiled build (-lineinfo) for nvdisasm -g."""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, obj, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
data = rows[2:]
iadr, iex, ist = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = int(data[0][iadr], 16)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = glob.glob(os.path.join(d, "*.cubin"))[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
# find the function section
lines = dis.splitlines()
fn_start = None
for i, l in enumerate(lines):
    if l.startswith(".text.") and kern in l:
        fn_start = i
        break
cur_line = None
off2line = {}
for l in lines[fn_start + 1:]:
    if l.startswith(".text.") or l.startswith("\t.section") and ".text." in l:
        break
    m = re.search(r'line (\d+)', l)
    if "//##" in l and m:
        mf = re.search(r'File "([^"]+)"', l)
        cur_line = (os.path.basename(mf.group(1)) if mf else "?", int(m.group(1)))
    m2 = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m2 and cur_line is not None:
        off2line[int(m2.group(1), 16)] = cur_line
ex = defaultdict(int)
st = defaultdict(int)
for r in data:
    off = int(r[iadr], 16) - base
    ln = off2line.get(off, ("?", -1))
    ex[ln] += int(r[iex] or 0)
    st[ln] += int(r[ist] or 0)
te, ts = sum(ex.values()), sum(st.values())
csrc = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2504_14611_b200", "csrc")
srcs = {}


def code_of(f, n):
    if f not in srcs:
        pth = os.path.join(csrc, f)
        srcs[f] = open(pth).read().splitlines() if os.path.exists(pth) else []
    L = srcs[f]
    return L[n - 1].strip()[:64] if 0 < n <= len(L) else "?"


print(f"total warp instructions {te:.4e}, stall samples {ts}")
for ln, s in sorted(st.items(), key=lambda x: -x[1])[:top]:
    f, n = ln
    print(f"{f[:16]:>16}:{n:<5d} stall {100*s/ts:5.1f}%  instr {100*ex[ln]/te:5.1f}%  {code_of(f, n)}")
