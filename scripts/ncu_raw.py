"""Key metrics of an `ncu -i X.ncu-rep --page raw --csv` export (one row per profiled kernel)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "smsp__inst_executed_pipe_fp64.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size"]
keys += [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled") or
         (h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"))]
for d in data:
    print("==", d[hdr.index("Kernel Name")][:90])
    vals = []
    for k in keys:
        if k in hdr:
            v = d[hdr.index(k)]
            try:
                fv = float(v.replace(",", ""))
            except ValueError:
                continue
            if k.startswith("smsp__pcsamp") and fv < 0.02 * max(1.0, fv) and fv == 0:
                continue
            vals.append((k, v, units[hdr.index(k)]))
    for k, v, u in vals:
        print(f"  {k:75s} {v} {u}")
