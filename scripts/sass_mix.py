"""Instruction mix of the innermost loops of a kernel containing a marker opcode (default
FFMA2): python scripts/sass_mix.py <binary> <function-substring> [marker]"""
import re
import subprocess
import sys
from collections import Counter

binary, fsub = sys.argv[1], sys.argv[2]
marker = sys.argv[3] if len(sys.argv) > 3 else "FFMA2"
out = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if fsub not in name:
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    # backward branches define loops [target, branch]
    loops = []
    for addr, txt in ins:
        m = re.search(r"BRA[^ ]* (?:[!]?U?P\d+, )?`?\(?0x([0-9a-f]+)", txt)
        if m:
            tgt = int(m.group(1), 16)
            if tgt <= addr:
                body = [t for a, t in ins if tgt <= a <= addr]
                if any(marker in t for t in body):
                    loops.append((tgt, addr, body))
    loops.sort(key=lambda l: l[1] - l[0])
    print(name)
    for tgt, addr, body in loops[:3]:
        ops = Counter()
        for t in body:
            t = re.sub(r"^@!?U?P[T0-9]+\s+", "", t)
            ops[t.split()[0].split(".")[0]] += 1
        print(f"  loop 0x{tgt:x}-0x{addr:x}: {len(body)} instr: " + ", ".join(f"{k} {v}" for k, v in ops.most_common()))
