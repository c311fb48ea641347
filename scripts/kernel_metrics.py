"""Per-kernel roofline evidence table (SURVEY §8(d) ncu list) from `ncu --set full` reports:
FMA-pipe instruction and cycle activity, XU (MUFU) pipe, DRAM bytes and throughput, shared-memory
bank conflicts, occupancy, issue activity.

    python scripts/kernel_metrics.py report.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma inst %pk"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma cyc %pk"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu inst %pk"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "issue %pk"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram %pk"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(m for m, _ in METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    print(f"# {rep}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        cells = [f"{lab}={d.get(m, '?')}{u.get(m, '')}" for m, lab in METRICS if m in d]
        print(f"{name:40s} grid={d.get('Grid Size', '?')} block={d.get('Block Size', '?')}  " + "  ".join(cells))
