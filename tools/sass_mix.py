"""Opcode histogram of a SASS address range: sass_mix.py file.sass START END (hex)."""
import re
import sys
from collections import Counter

path, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
cnt = Counter()
for line in open(path):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and lo <= int(m.group(1), 16) < hi:
        cnt[m.group(3)] += 1
tot = sum(cnt.values())
print("total", tot)
for k, v in cnt.most_common(30):
    print(f"{v:5d} {k}")
