"""List the backward-branch loops of a kernel in a cuobjdump -sass dump (size in instructions,
and whether the body holds a marker opcode).  python scripts/sass_loops.py dump.sass kernel_substr [marker]"""
import re, sys
lines = open(sys.argv[1]).read().split('\n')
funcs, cur = {}, None
for l in lines:
    m = re.search(r'Function : (\S+)', l)
    if m:
        cur = m.group(1); funcs[cur] = []; continue
    if cur and re.match(r'\s+/\*[0-9a-f]{4,5}\*/', l):
        funcs[cur].append(l)
name = [f for f in funcs if sys.argv[2] in f][0]
body = funcs[name]
addr = [int(l.split('/*')[1].split('*/')[0], 16) for l in body]
marker = sys.argv[3] if len(sys.argv) > 3 else None
print(name, len(body), "instructions")
for i, l in enumerate(body):
    m = re.search(r'BRA (0x[0-9a-f]+)', l)
    if m and int(m.group(1), 16) < addr[i]:
        lo = int(m.group(1), 16)
        seg = [b for b, a in zip(body, addr) if lo <= a <= addr[i]]
        has = any(marker in b for b in seg) if marker else ""
        print(f"loop {lo:#x}-{addr[i]:#x}: {len(seg)} instructions {has}")
