"""Key counters of an `ncu --set full` capture (one launch per report section):
python tools/ncu_full_summary.py report.ncu-rep > profiles/<tag>_summary.txt"""
import csv
import subprocess
import sys

SECTION = ("DRAM Frequency", "SM Frequency", "Elapsed Cycles", "Memory Throughput", "DRAM Throughput", "Duration",
           "L1/TEX Cache Throughput", "L2 Cache Throughput", "SM Active Cycles", "Compute (SM) Throughput",
           "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate", "Block Size", "Cluster Size", "Grid Size",
           "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
       "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio")


def rows(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


rep = sys.argv[1]
det = rows(rep, "details")
hdr = det[0]
seen = set()
for r in det[1:]:
    d = dict(zip(hdr, r))
    if "Kernel Name" in d and d["ID"] not in seen:
        seen.add(d["ID"])
        print(f"kernel: {d['Kernel Name']} grid {d.get('Grid Size', '')} block {d.get('Block Size', '')}")
    if d.get("Metric Name") in SECTION:
        print(f"{d['Metric Name']:45s} {d['Metric Value']} {d['Metric Unit']}")
raw = rows(rep, "raw")
h = raw[0]
for r in raw[2:]:
    d = dict(zip(h, r))
    for k in RAW:
        if k in d:
            print(f"{k:90s} {d[k]}")
