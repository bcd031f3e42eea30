"""List the loops (backward branches) of one kernel's SASS with their
instruction mix.  usage: cuobjdump -sass lib.so | python tools/sass_loops.py <mangled-substring>"""
import collections
import re
import sys

want = sys.argv[1]
code, on = [], False
for line in sys.stdin:
    if "Function :" in line:
        on = want in line
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if on and m:
        code.append((int(m.group(1), 16), m.group(2).strip()))
for addr, ins in code:
    m = re.search(r"BRA (?:\S+, )?0x([0-9a-f]+)", ins)
    if m and int(m.group(1), 16) < addr:
        tgt = int(m.group(1), 16)
        body = [i for a, i in code if tgt <= a <= addr]
        if len(body) < 40:
            continue
        ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", i).split()[0].split(".")[0] for i in body)
        print(f"loop {tgt:#x}-{addr:#x} n={len(body)}: " + " ".join(f"{k}:{v}" for k, v in ops.most_common(12)))
