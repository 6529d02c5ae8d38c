"""Condense an `ncu --page details --csv` dump into the summary lines kept
under profiles/ (dev aid): python scripts/ncu_summary.py details.csv [report.ncu-rep]"""
import csv, io, subprocess, sys
KEEP = {
    ("GPU Speed Of Light Throughput", "Memory Throughput"), ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "Duration"), ("GPU Speed Of Light Throughput", "L1/TEX Cache Throughput"),
    ("GPU Speed Of Light Throughput", "L2 Cache Throughput"), ("Compute Workload Analysis", "Executed Ipc Active"),
    ("Compute Workload Analysis", "Issue Slots Busy"), ("Memory Workload Analysis", "Memory Throughput"),
    ("Memory Workload Analysis", "L1/TEX Hit Rate"), ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Scheduler Statistics", "Active Warps Per Scheduler"), ("Scheduler Statistics", "Eligible Warps Per Scheduler"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"), ("Warp State Statistics", "Avg. Active Threads Per Warp"),
    ("Launch Statistics", "Block Size"), ("Launch Statistics", "Grid Size"), ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Dynamic Shared Memory Per Block"), ("Launch Statistics", "Static Shared Memory Per Block"),
    ("Occupancy", "Theoretical Occupancy"), ("Occupancy", "Achieved Active Warps Per SM"),
}
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value")}
seen = None
for r in rows[hi + 1:]:
    if len(r) <= ix["Metric Value"]:
        continue
    if r[ix["ID"]] != seen:
        seen = r[ix["ID"]]
        print(f"## launch {seen}: {r[ix['Kernel Name']][:90]}")
    if (r[ix["Section Name"]], r[ix["Metric Name"]]) in KEEP:
        print(f"{r[ix['Section Name']]:30s} {r[ix['Metric Name']]:40s} {r[ix['Metric Value']]} {r[ix['Metric Unit']]}")
if len(sys.argv) > 2:
    raw = subprocess.run(["ncu", "-i", sys.argv[2], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh = rr[0]
    for row in rr[2:]:
        d = dict(zip(hh, row))
        out = []
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                  "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
                  "gpu__time_duration.sum"):
            if k in d:
                out.append(f"{k} {d[k]} {rr[1][hh.index(k)]}")
        print("; ".join(out))
