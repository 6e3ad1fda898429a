"""Stall reasons and headline metrics of every kernel in an ncu report.  usage: ncu_stalls.py report.ncu-rep"""
import csv, subprocess, sys, io
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    print("==", d.get("Kernel Name", "?")[:70], "dur(us)", d.get("gpu__time_duration.sum"))
    items = []
    for k, x in d.items():
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("_not_issued"):
            try: items.append((float(x.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError: pass
    s = sum(i[0] for i in items) or 1
    print("  stalls:", ", ".join(f"{k} {val / s * 100:.0f}%" for val, k in sorted(items, reverse=True)[:7]))
    for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
              "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
              "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_op_write.sum", "lts__t_sector_hit_rate.pct"]:
        if k in d: print(f"  {k} = {d[k]}")
