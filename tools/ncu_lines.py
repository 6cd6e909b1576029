"""Aggregate ncu source-page warp-stall samples per CUDA source line.
usage: python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top]"""
import csv, subprocess, sys, collections, re
rep = sys.argv[1]; kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"]
if kre: cmd += ["-k", "regex:" + kre]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = None; hdr = None; agg = collections.Counter(); src = {}; total = 0
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or not r[0].isdigit(): continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    try: v = float(r[si] or 0)
    except ValueError: continue
    key = (cur_file, int(r[0])); agg[key] += v; total += v
    src[key] = r[1].strip()[:90]
for (f, l), v in agg.most_common(top):
    print(f"{v/total:6.1%} {f}:{l:<5d} {src[(f,l)]}")
