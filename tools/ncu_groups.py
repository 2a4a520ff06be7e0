"""Samples / executed instructions of an ncu source page grouped by code region:
    ncu -i REP --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_groups.py src.csv"""
import csv
import sys

G = [("kernels.cuh", 307, 334, "band1_terms (cached terms)"),
     ("kernels.cuh", 239, 299, "band1 (dense band, own diff)"), ("kernels.cuh", 151, 222, "band"),
     ("kernels.cuh", 341, 414, "edges"), ("kernels.cuh", 418, 452, "band_generic"),
     ("kernels.cuh", 453, 586, "diff windows"), ("kernels.cuh", 587, 771, "station_item setup"),
     ("kernels.cuh", 772, 804, "arrival_item"), ("kernels.cuh", 805, 840, "score_item dispatch"),
     ("kernels.cuh", 1, 150, "kernels.cuh helpers (term, warp_sum, cp.async)"),
     ("seis_philox.h", 1, 400, "philox + Box-Muller"), ("engine.cuh", 278, 287, "make_win"),
     ("engine.cuh", 296, 299, "inw"), ("engine.cuh", 288, 295, "yix/pix"),
     ("engine.cuh", 306, 313, "arrival_mean / div_v"), ("engine.cuh", 314, 336, "ver_arr / arr_of"),
     ("engine.cuh", 337, 350, "arr_logpdf"), ("phase.cuh", 485, 640, "tile-major loop"),
     ("phase.cuh", 641, 713, "proposal-major loop"), ("phase.cuh", 16, 205, "gen_proposal"),
     ("phase.cuh", 206, 412, "k_phase prologue"), ("phase.cuh", 413, 484, "round head"),
     ("phase.cuh", 714, 1015, "decision"), ("phase.cuh", 1016, 1102, "write-back"),
     ("phase.cuh", 1103, 1200, "phase outputs")]
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
