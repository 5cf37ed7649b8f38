"""Print the headline metrics of one ncu report (read here, no GPU)."""
import csv
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue%"),
    ("smsp__inst_executed.sum", "inst"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
]
STALL = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio"
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2]
    print("==", rep, v[h.index("Kernel Name")][:80] if "Kernel Name" in h else "")
    print("  " + "  ".join(f"{n}={v[h.index(m)]}" for m, n in WANT if m in h))
    st = []
    for m in h:
        if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[h.index(m)]), m[34:-23]))
            except ValueError:
                pass
    st.sort(reverse=True)
    print("  stalls: " + " ".join(f"{n}={x:.2f}" for x, n in st[:8]))
