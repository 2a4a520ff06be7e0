"""Top source lines of an ncu source page by one stall reason:
    python tools/ncu_stall_lines.py src.csv stall_long_sb [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
col = sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
f, hdr, out, tot = None, None, [], 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d[col])
    except (ValueError, KeyError):
        continue
    tot += s
    out.append((s, f, int(r[0]), r[1][:100]))
out.sort(reverse=True)
print(f"total {col} samples {tot}")
for s, f, ln, src in out[:n]:
    print(f"{100 * s / max(tot, 1):5.1f}% {f}:{ln} {src}")
