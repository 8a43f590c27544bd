"""Summarise an ncu --set full report (one kernel launch) into the text
files kept under profiles/: duration, instruction count, IPC, occupancy,
registers, DRAM bytes and the warp-stall breakdown.
usage: python profiles/ncu_summary.py report.ncu-rep > profiles/rNN_cX_ncu_summary.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
for v in rows[2:]:
    print("kernel", v[h.index("Kernel Name")])
    for w in ["gpu__time_duration.sum", "smsp__inst_executed.sum",
              "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
              "launch__grid_size", "launch__block_size",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "smsp__thread_inst_executed_per_inst_executed.ratio",
              "sm__cycles_elapsed.avg.per_second"]:
        if w in h:
            i = h.index(w)
            print("   %-55s %s %s" % (w, v[i], units[i]))
    st = []
    for i, x in enumerate(h):
        if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued"):
            try:
                st.append((float(v[i]), x.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in st) or 1.0
    for s, n in sorted(st, reverse=True)[:10]:
        print("   stall %5.1f%% %s" % (100 * s / tot, n))
