"""Samples / executed instructions of an ncu source page grouped by code region:
    ncu -i REP --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_groups.py src.csv"""
import csv
import sys

import os
import re

CSRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1612_00595_b200", "csrc")
# (file, first line of the region as a regex, label): a region runs to the next marker of its file
MARKS = [
    ("kernels.cuh", r"^struct Y2;", "kernels.cuh helpers (term, warp_sum)"),
    ("kernels.cuh", r"void band\(const Dev", "band (generic rows)"),
    ("kernels.cuh", r"void band1\(const Dev", "band1 (dense band, own diff)"),
    ("kernels.cuh", r"void band1_terms\(", "band1_terms (cached terms)"),
    ("kernels.cuh", r"void dense_pair_terms\(", "dense_pair_terms (tile pairs, cached terms)"),
    ("kernels.cuh", r"void edges\(const Dev", "edges"),
    ("kernels.cuh", r"void band_generic\(", "band_generic"),
    ("kernels.cuh", r"^struct DiffW", "diff windows"),
    ("kernels.cuh", r"void station_item\(", "station_item setup"),
    ("kernels.cuh", r"void arrival_item\(", "arrival_item"),
    ("kernels.cuh", r"void score_item\(", "score_item dispatch"),
    ("engine.cuh", r"Win make_win\(", "make_win"),
    ("engine.cuh", r"size_t yix\(", "yix/pix"),
    ("engine.cuh", r"int inw\(", "inw"),
    ("engine.cuh", r"double div_v\(", "arrival_mean / div_v"),
    ("engine.cuh", r"double gen_arrival\(", "ver_arr / arr_of"),
    ("engine.cuh", r"double arr_logpdf\(", "arr_logpdf"),
    ("phase.cuh", r"^__device__ void gen_proposal", "gen_proposal"),
    ("phase.cuh", r"k_phase\(const Dev d", "k_phase prologue"),
    ("phase.cuh", r"for \(int i0 = 0; i0 < \(int\)sp.k; \+\+round\)", "round head"),
    ("phase.cuh", r"if constexpr \(TM\) \{", "tile-major loop"),
    ("phase.cuh", r"int cur_q = -1;", "proposal-major loop"),
    ("phase.cuh", r"// S2: partial sums ready", "decision"),
    ("phase.cuh", r"// S3: decision", "write-back"),
    ("phase.cuh", r"// ---- phase outputs", "phase outputs"),
]


def build_groups():
    out = []
    by_file = {}
    for f, rx, label in MARKS:
        by_file.setdefault(f, []).append((rx, label))
    for f, marks in by_file.items():
        path = os.path.join(CSRC, f)
        if not os.path.exists(path):
            continue
        lines = open(path).read().split("\n")
        starts = []
        for rx, label in marks:
            for i, line in enumerate(lines, 1):
                if re.search(rx, line):
                    starts.append((i, label))
                    break
        starts.sort()
        for k, (ln, label) in enumerate(starts):
            # a function's template / comment header sits just above its first line
            hi = starts[k + 1][0] - 1 if k + 1 < len(starts) else len(lines)
            out.append((f, ln, hi, label))
    out.append(("seis_philox.h", 1, 100000, "philox + Box-Muller"))
    return out


G = build_groups()
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
