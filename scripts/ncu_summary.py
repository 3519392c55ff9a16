"""Summarise an ncu report (--page raw --csv) into the key counters (one kernel per row)."""
import csv, subprocess, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
STALLS = ["wait", "short_scoreboard", "long_scoreboard", "barrier", "mio_throttle", "math_pipe_throttle",
          "lg_throttle", "not_selected", "selected", "dispatch_stall", "no_instruction", "membar", "drain",
          "branch_resolving", "tex_throttle", "sleeping", "misc"]
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print(f"== {rep}: {v[h.index('Kernel Name')][:90]}")
        for k in KEYS:
            if k in h:
                print(f"  {k:70s} {v[h.index(k)]} {units[h.index(k)]}")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in h:
                st.append(f"{s}={float(v[h.index(k)]):.2f}")
        print("  stalls/issue: " + " ".join(st))
