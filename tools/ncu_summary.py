"""Summarise one kernel of an ncu --set full report (.ncu-rep) into metric,value,unit CSV lines.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep k_syrk > profiles/rNN_ncu_syrk_tc_summary.csv
"""
import csv
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
           "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__cluster_dim_x", "launch__grid_size", "launch__block_size"]


def main(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kernel}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    print("metric,value,unit")
    for m in METRICS:
        if m in h:
            i = h.index(m)
            print(f"{m},{v[i].replace(',', '')},{u[i]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
