"""Summarise an ncu --set full report (raw page CSV) into the metrics we track.

    ncu -i prof.ncu-rep --page raw --csv > raw.csv && python profiles/ncu_summary.py raw.csv
"""
import csv
import sys

WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
]


def main(path):
    rows = list(csv.reader(open(path)))
    h, units, data = rows[0], rows[1], rows[2:]
    name_i = h.index("Kernel Name")
    for r in data:
        print(f"== {r[name_i][:90]}")
        for w in WANT:
            hits = [i for i, x in enumerate(h) if x == w]
            if not hits:
                hits = [i for i, x in enumerate(h) if x.startswith(w.split(".")[0]) and "pct" in x and w.split(".")[0] in ("sm__pipe_tensor_cycles_active",)]
            for i in hits[:1]:
                print(f"   {w:70s} {r[i]:>18s} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
