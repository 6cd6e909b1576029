"""Per-kernel SASS mnemonic counts of the product library (evidence that the
hot kernels issue the intended instructions: DMMA for the fp64 train step,
UTCHMMA / UTCQMMA + UTMALDG + LDTM for the tcgen05 GEMMs, FFMA2 for inference).
usage: python tools/sass_summary.py [lib.so] > profiles/<round>/sass_summary.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2111_12055_b200/libgbxcu.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
KEYS = ["DMMA", "DFMA", "DADD", "DMUL", "FFMA2", "FFMA", "HMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG",
        "UTMASTG", "LDTM", "STTM", "LDGSTS", "LDGDEPBAR", "SHFL", "BAR", "MEMBAR", "RED", "ATOMS", "LDS", "STS"]
kern = None
counts = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    if kern is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m:
        op = m.group(1)
        counts[kern][op] += 1
        counts[kern]["_total"] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


names = list(counts)
pretty = demangle(names)
print("# SASS mnemonic counts per kernel (`cuobjdump -sass " + lib + "`)\n")
print("| kernel | instr | " + " | ".join(KEYS) + " |")
print("|---" * (len(KEYS) + 2) + "|")
for n, p in sorted(zip(names, pretty), key=lambda x: x[1]):
    c = counts[n]
    if not any(c[k] for k in KEYS):
        continue
    short = re.sub(r"\(.*", "", p.replace("gbxcu::", "")).replace("(anonymous namespace)::", "")
    print(f"| `{short[:70]}` | {c['_total']} | " + " | ".join(str(c[k]) if c[k] else "" for k in KEYS) + " |")
