"""Summarise an ncu --set full report (raw page) into the metrics the design cares about.

Usage: python scripts/ncu_summary.py REPORT.ncu-rep [--json OUT.json --config P --variant NAME]
"""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2:]
want = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
]
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
out = []
for v in vals:
    d = {}
    for w in want + stalls:
        if w in hdr:
            i = hdr.index(w)
            d[w] = (v[i], units[i])
    out.append(d)
for d in out:
    for k, (v, u) in d.items():
        try:
            if k in stalls and float(v.replace(",", "")) < 0.05:
                continue
        except ValueError:
            pass
        print(f"{k:80s} {v:>22s} {u}")
    print()
if "--json" in sys.argv and out:
    d = out[0]
    f = lambda k: float(d[k][0].replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(d[k][1], 1.0)
    j = {
        "config": sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else None,
        "variant": sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else None,
        "source": rep,
        "dram_read_bytes": f("dram__bytes_read.sum"),
        "dram_write_bytes": f("dram__bytes_write.sum"),
        "dram_bytes_per_launch": f("dram__bytes_read.sum") + f("dram__bytes_write.sum"),
        "lts_sector_hit_rate_pct": float(d["lts__t_sector_hit_rate.pct"][0]),
        "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
        "inst_executed": float(d["smsp__inst_executed.sum"][0].replace(",", "")),
        "duration_ms_under_ncu": float(d["gpu__time_duration.sum"][0]) * (1e-3 if d["gpu__time_duration.sum"][1] == "us" else 1.0),
    }
    with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
        json.dump(j, fh, indent=1)
