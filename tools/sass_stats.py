"""Static SASS opcode histogram per kernel of libfllf.so (quick check of FFMA2 use / MOV overhead)."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2206_04681_b200/lib/libfllf.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, stats = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        k = re.search(r"(k_\w+?)I(\w+?)EEvNS", name)
        cur = (k.group(1) + "<" + k.group(2) + ">") if k else name
        stats[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        stats[cur][m.group(2)] += 1
for k, c in stats.items():
    tot = sum(c.values())
    top = ", ".join(f"{op}:{n}" for op, n in c.most_common(12))
    print(f"{k:40s} total {tot:5d}  {top}")
