"""Top source lines of an ncu report by warp-stall samples:
    ncu -i REP --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
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
    if hdr is None or r[0] == "Function Name" or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"])
        ins = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    tot += s
    out.append((s, ins, f, int(r[0]), r[1][:90]))
out.sort(reverse=True)
print(f"total samples {tot}")
for s, ins, f, ln, src in out[:n]:
    print(f"{100 * s / tot:5.1f}% {ins / 1e6:8.1f}M {f}:{ln} {src}")


def by_range(path, ranges):
    """sum samples / executed instructions over (file, lo, hi, name) ranges"""
    rows = list(csv.reader(open(path)))
    f, hdr = None, None
    acc = {r[3]: [0, 0] for r in ranges}
    tot = [0, 0]
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
            s = int(d["Warp Stall Sampling (All Samples)"])
            ins = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        tot[0] += s
        tot[1] += ins
        ln = int(r[0])
        for (ff, lo, hi, name) in ranges:
            if ff == f and lo <= ln <= hi:
                acc[name][0] += s
                acc[name][1] += ins
                break
    for name, (s, ins) in acc.items():
        print(f"{name:28s} samples {100 * s / tot[0]:5.1f}%  instr {100 * ins / tot[1]:5.1f}%")
    print(f"total instr {tot[1] / 1e9:.2f} G")
