"""Summarise an ncu report (raw page) into the metrics the design cares about; optional JSON output."""
import csv, io, json, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
        "smsp__inst_executed.avg.per_cycle_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__average_warp_latency_issue_stalled_short_scoreboard",
        "smsp__average_warp_latency_issue_stalled_barrier", "smsp__average_warp_latency_issue_stalled_membar",
        "smsp__average_warp_latency_issue_stalled_mio_throttle", "smsp__average_warp_latency_issue_stalled_lg_throttle",
        "smsp__average_warp_latency_issue_stalled_wait", "smsp__average_warp_latency_issue_stalled_no_instruction",
        "smsp__average_warp_latency_issue_stalled_math_pipe_throttle", "smsp__average_warp_latency_issue_stalled_dispatch_stall",
        "smsp__average_warp_latency_issue_stalled_not_selected", "smsp__average_warp_latency_issue_stalled_selected",
        "smsp__average_warp_latency_issue_stalled_branch_resolving", "smsp__average_warp_latency_issue_stalled_drain",
        "smsp__average_warp_latency_issue_stalled_imc_miss", "smsp__average_warp_latency_issue_stalled_sleeping",
        "smsp__warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "smsp__warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__warps_issue_stalled_mio_throttle_per_issue_active.ratio", "smsp__warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__warps_issue_stalled_barrier_per_issue_active.ratio", "smsp__warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "smsp__warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__warps_issue_stalled_no_instruction_per_issue_active.ratio", "smsp__warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "smsp__warps_issue_stalled_selected_per_issue_active.ratio"]
out = []
for v in vals:
    d = {}
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            d[w] = (v[i], units[i])
    out.append(d)
for d in out:
    for k, (v, u) in d.items():
        print(f"{k:75s} {v:>22s} {u}")
    print()
