"""Samples / executed instructions of an ncu source page grouped by code region:
    ncu -i REP --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_groups.py src.csv"""
import csv
import sys

G = [("kernels.cuh", 226, 285, "band1 (dense band)"), ("kernels.cuh", 138, 209, "band"),
     ("kernels.cuh", 293, 365, "edges"), ("kernels.cuh", 369, 403, "band_generic"),
     ("kernels.cuh", 405, 527, "diff windows"), ("kernels.cuh", 529, 700, "station_item setup"),
     ("kernels.cuh", 700, 735, "arrival_item"), ("kernels.cuh", 735, 760, "score_item dispatch"),
     ("kernels.cuh", 1, 137, "kernels.cuh helpers (term, warp_sum)"),
     ("seis_philox.h", 1, 400, "philox + Box-Muller"), ("engine.cuh", 245, 253, "make_win"),
     ("engine.cuh", 263, 265, "inw"), ("engine.cuh", 255, 262, "yix/pix"),
     ("engine.cuh", 273, 280, "arrival_mean / div_v"), ("engine.cuh", 282, 302, "ver_arr / arr_of"),
     ("engine.cuh", 304, 314, "arr_logpdf"), ("engine.cu", 686, 743, "tile-major loop"),
     ("engine.cu", 744, 811, "proposal-major loop"), ("engine.cu", 234, 423, "gen_proposal"),
     ("engine.cu", 424, 620, "k_phase prologue"), ("engine.cu", 621, 685, "round head"),
     ("engine.cu", 812, 1115, "decision"), ("engine.cu", 1116, 1200, "write-back"),
     ("engine.cu", 1200, 1290, "phase outputs")]
rows = list(csv.reader(open(sys.argv[1])))
f, hdr = None, None
acc = {g[3]: [0, 0] for g in G}
acc["other"] = [0, 0]
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
    except (ValueError, KeyError):
        continue
    ln = int(r[0])
    name = "other"
    for g in G:
        if g[0] == f and g[1] <= ln <= g[2]:
            name = g[3]
            break
    acc[name][0] += s
    acc[name][1] += ins
    tot[0] += s
    tot[1] += ins
print(f"total samples {tot[0]}, instructions {tot[1] / 1e9:.2f} G")
for k, (s, i) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    if s or i:
        print(f"{100 * s / tot[0]:5.1f}% samples  {100 * i / max(tot[1], 1):5.1f}% instr  {i / 1e6:9.1f}M  {k}")
