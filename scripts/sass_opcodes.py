"""Per-kernel counts of the Blackwell opcodes that prove the tcgen05 / TMA / packed-FP32 paths,
from cuobjdump -sass of the built librici.so (static instruction counts, not executions).
    python scripts/sass_opcodes.py [librici.so] > profiles/r2_sass_opcodes.txt"""
import collections, re, subprocess, sys, os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2007_02306_b200", "librici.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
WANT = ["UTCIMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "UTCCP", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM",
        "SYNCS", "FFMA2", "FADD2", "FMUL2", "ATOMS", "REDS", "MUFU", "IDP", "VOTE", "SHFL"]
kern, counts = None, collections.defaultdict(collections.Counter)
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        kern = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
    if kern and m:
        op, mods = m.group(1), m.group(2) or ""
        for w in WANT:
            if op == w:
                counts[kern][op + (mods if w in ("UTCIMMA", "UTMALDG", "UTCBAR", "UTCCP") else "")] += 1
                counts[kern]["_" + op] += 1
print(f"# static SASS opcode counts per kernel, cuobjdump -sass {os.path.relpath(lib, ROOT)} (sm_100a)")
for k in sorted(counts):
    c = counts[k]
    short = re.sub(r"_ZN4rici\d*(_GLOBAL__N__\w+?_\d+)?", "", k)[:90]
    items = ", ".join(f"{op}={n}" for op, n in sorted(c.items()) if not op.startswith("_"))
    print(f"{short}\n    {items}")
