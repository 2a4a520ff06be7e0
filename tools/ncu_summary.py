"""Markdown summary of one k_phase launch from an ncu --set full report:
    ncu -i REP --page raw --csv > raw.csv
    ncu -i REP --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_summary.py raw.csv src.csv > profiles/rNN_ncu_k_phase_configX.md"""
import csv
import subprocess
import sys

raw, src = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(raw)))
h, u, v = rows[0], rows[1], rows[2]
m = {name: (v[i], u[i]) for i, name in enumerate(h)}


def g(name, fmt="{:.3g}", scale=1.0):
    if name not in m:
        return "n/a"
    try:
        return fmt.format(float(m[name][0].replace(",", "")) * scale) + " " + m[name][1]
    except ValueError:
        return m[name][0]


print("| metric | value |\n|---|---|")
for label, name, fmt in [
        ("kernel", "Kernel Name", None), ("grid x block", "Grid Size", None),
        ("duration (under ncu: cold caches, serialised)", "gpu__time_duration.sum", "{:.2f}"),
        ("dram read", "dram__bytes_read.sum", "{:.2f}"), ("dram write", "dram__bytes_write.sum", "{:.2f}"),
        ("L2 sectors read from L1/tex (x 32 B)", "lts__t_sectors_srcunit_tex_op_read.sum", "{:.4g}"),
        ("L2 hit rate", "lts__t_sector_hit_rate.pct", "{:.1f}"),
        ("L1 hit rate", "l1tex__t_sector_hit_rate.pct", "{:.1f}"),
        ("L1/LSU data pipe throughput", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "{:.1f}"),
        ("instructions (warp)", "smsp__inst_executed.sum", "{:.4g}"),
        ("issue slots busy", "smsp__issue_active.avg.pct_of_peak_sustained_active", "{:.1f}"),
        ("warps active", "sm__warps_active.avg.pct_of_peak_sustained_active", "{:.1f}"),
        ("registers per thread", "launch__registers_per_thread", "{:.0f}"),
        ("SM active cycles mean", "sm__cycles_active.avg", "{:.4g}"), ("SM active cycles max", "sm__cycles_active.max", "{:.4g}"),
        ("pipe ALU", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "{:.1f}"),
        ("pipe FMA (fp32)", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "{:.1f}"),
        ("pipe FP64", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "{:.1f}"),
        ("pipe XU (SFU)", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "{:.1f}"),
        ("pipe LSU", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "{:.1f}")]:
    if name in m:
        print(f"| {label} | {m[name][0] if fmt is None else g(name, fmt)} |")
print("\nStalls per issued instruction (warps per scheduler waiting, by reason):\n")
st = []
for name in h:
    if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(m[name][0]), name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
st.sort(reverse=True)
tot = sum(x for x, _ in st) or 1.0
print(", ".join(f"{n} {x:.2f} ({100 * x / tot:.0f} %)" for x, n in st[:9]))
print("\nBy code region (pc samples, executed warp instructions):\n\n```")
print(subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_groups.py"), src],
                     capture_output=True, text=True).stdout.strip())
print("```\n\nLong-scoreboard stalls by source line:\n\n```")
print(subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_stall_lines.py"), src,
                      "stall_long_sb", "8"], capture_output=True, text=True).stdout.strip())
print("```")
