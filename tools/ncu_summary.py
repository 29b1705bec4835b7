"""Summarise ncu --set full reports: one CSV row per launch with the metrics the design
claims rest on (time, DRAM bytes, tensor-pipe activity, SM / memory throughput, regs).

    python tools/ncu_summary.py REPORT.ncu-rep [...] > profiles/<name>.csv
"""
import csv, io, subprocess, sys

KEEP = [
    ("Kernel Name", "kernel"),
    ("Grid Size", "grid"),
    ("Block Size", "block"),
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    # tcgen05 activity: busy fraction of the SM's tensor-core (TMEM-side) datapath
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tcgen05_active_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_throughput_pct"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_tc_wavefronts_pct"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("launch__registers_per_thread", "regs"),
]
w = csv.writer(sys.stdout)
w.writerow(["report"] + [k for _, k in KEEP])
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    w.writerow(["(units)"] + [units[idx[m]] if m in idx else "" for m, _ in KEEP])
    for r in rows[2:]:
        w.writerow([rep.split("/")[-1]] + [r[idx[m]] if m in idx else "" for m, _ in KEEP])
