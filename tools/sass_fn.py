"""Extract one function's SASS from `cuobjdump -sass` output and count
opcodes.  Usage: python tools/sass_fn.py all.sass <name substring> [--dump]"""
import re
import sys
from collections import Counter

text = open(sys.argv[1]).read()
key = sys.argv[2]
parts = re.split(r"\n\s*Function : ", text)
for part in parts[1:]:
    name = part.split("\n", 1)[0].strip()
    if key in name:
        body = part.split("\n", 1)[1]
        ops = Counter()
        for line in body.splitlines():
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
            if m:
                ops[m.group(1)] += 1
        print(name, sum(ops.values()), "instructions")
        print("  ", ", ".join(f"{k}={v}" for k, v in ops.most_common(24)))
        if "--dump" in sys.argv:
            print(body)
