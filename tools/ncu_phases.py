"""Attribute ncu warp-stall samples of a kernel to the '// ---- <phase>' blocks of
its source file. usage: python tools/ncu_phases.py report.ncu-rep kernel-regex file.cu"""
import collections, re, subprocess, sys
rep, kre, src = sys.argv[1], sys.argv[2], sys.argv[3]
lines = open(src).read().splitlines()
marks = [(i + 1, re.sub(r"\s+", " ", l.strip()[8:48])) for i, l in enumerate(lines) if l.strip().startswith("// ---- ")]
def phase(ln):
    name = "(prologue/other)"
    for start, nm in marks:
        if ln >= start: name = nm
    return name
out = subprocess.run(["python", "tools/ncu_lines.py", rep, kre, "100000"], capture_output=True, text=True).stdout
agg = collections.Counter(); other = collections.Counter()
fname = src.split("/")[-1]
for l in out.splitlines():
    m = re.match(r"\s*([\d.]+)% (\S+):(\d+)", l)
    if not m: continue
    v, f, ln = float(m.group(1)), m.group(2), int(m.group(3))
    if f == fname: agg[phase(ln)] += v
    else: other[f] += v
for k, v in agg.most_common(): print(f"{v:6.1f}%  {k}")
for k, v in other.most_common(): print(f"{v:6.1f}%  [{k}]")
