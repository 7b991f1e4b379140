"""Print the key sections of an `ncu --set full` report (details page) as text,
plus dram read/write bytes from the raw page.  Usage: summarize_ncu.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEEP = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy",
        "Launch Statistics", "Scheduler Statistics", "Warp State Statistics",
        "Compute Workload Analysis")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "sm__inst_executed_pipe_fp64.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor_subpipe_dmma.sum")


def main(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    hdr = rows[0]
    ki, si, mi, ui, vi = (hdr.index(h) for h in ("Kernel Name", "Section Name", "Metric Name",
                                                  "Metric Unit", "Metric Value"))
    kern = None
    for r in rows[1:]:
        if r[ki] != kern:
            kern = r[ki]
            print(f"== {kern}")
        if r[si] in KEEP and r[mi]:
            print(f"  {r[si][:28]:28s} {r[mi][:44]:44s} {r[vi]:>16s} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, u = rr[0], rr[1]
    for vals in rr[2:]:
        print("== raw", vals[h.index("Kernel Name")][:60])
        for name in RAW:
            if name in h:
                i = h.index(name)
                print(f"  {name:64s} {vals[i]:>18s} {u[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
