"""Summarise an ncu report (raw page) for the kernels of interest: time,
DRAM traffic, tensor-pipe utilisation, occupancy.  Usage:
  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [extra-metric-substring ...]"""
import csv, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__cycles_active.avg", "gpc__cycles_elapsed.max"]


def main():
    rep = sys.argv[1]
    extra = sys.argv[2:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    keys = KEYS + [h for h in hdr if any(e in h for e in extra)]
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")][:60]
        print("==", name)
        for k in keys:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {k:75s} {row[i]:>14s} {units[i]}")


if __name__ == "__main__":
    main()
