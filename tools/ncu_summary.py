"""Summarise an `ncu --page raw --csv` export: one block per profiled kernel."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]


def main(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[h.index("Kernel Name")][:110])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print("   %-66s %s %s" % (k, r[i], units[i]))
        stalls = [(float(r[i].replace(",", "") or 0), x) for i, x in enumerate(h)
                  if x.startswith("smsp__average_warp_latency_issue_stalled") and x.endswith(".ratio")]
        stalls.sort(reverse=True)
        print("   top stalls:", ", ".join("%s=%.2f" % (n.split("stalled_")[1].split(".")[0], v) for v, n in stalls[:6]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
