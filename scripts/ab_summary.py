"""Summarise scripts/ab_formats.py output: per (case, precision, G) the
variants ranked by their best back-to-back time (us)."""
import collections
import re
import sys

rows = collections.defaultdict(dict)
for line in open(sys.argv[1]):
    m = re.match(r'(\S+) p(\d)(?: g(\d+))? (\S+)\s+b2b us\s+([\d. ]+)\|\s*flushed us\s+([\d. ]+)', line)
    if m:
        c, p, g, v, b, f = m.groups()
        rows[(c, p, g or "32")][v] = (min(map(float, b.split())), min(map(float, f.split())))
    elif "NOT bitwise" in line:
        print(line.strip())
for k, d in rows.items():
    best = sorted(d.items(), key=lambda t: t[1][0])
    print(":".join(k), " ".join(f"{v}:{t[0]:.1f}" for v, t in best[:8]))
