"""Aggregate ncu source-page warp-stall samples per CUDA source line.
usage: python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top] [function-substring]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
fsub = sys.argv[4] if len(sys.argv) > 4 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"]
if kre: cmd += ["-k", "regex:" + kre]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = None; cur_fn = ""; hdr = None; agg = collections.Counter(); src = {}; total = 0
for r in rows:
    if not r: continue
    if r[0] in ("File Path", "File Name"): cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": cur_fn = r[1]; continue
    if r[0] == "Line No": hdr = r; continue
    if fsub and fsub not in cur_fn: continue
    if hdr is None or not r[0].isdigit(): continue
    try:
        si = hdr.index("Warp Stall Sampling (All Samples)")
        v = float(r[si] or 0)
    except (ValueError, IndexError):
        continue
    key = (cur_file, int(r[0])); agg[key] += v; total += v
    src.setdefault(key, r[1].strip()[:90])
for (f, l), v in agg.most_common(top):
    print(f"{v/max(total,1):6.1%} {f}:{l:<5d} {src[(f,l)]}")
