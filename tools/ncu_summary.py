"""Summarise an ncu report: key raw metrics + top stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "smsp__inst_executed_op_global_ld.sum", "smsp__inst_executed_op_global_st.sum",
        "sm__warps_active.avg.per_cycle_active"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print("kernel:", name[:100])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:70s} {v[i]} {units[i]}")
        stalls = [(float(v[i].replace(',', '')), h[i]) for i in range(len(h))
                  if h[i].startswith("smsp__average_warp_latency_issue_stalled") and
                  h[i].endswith(".ratio") and v[i] not in ("", "n/a")]
        stalls = sorted([s for s in stalls if s[0] > 0.05], reverse=True)[:8]
        for s, nm in stalls:
            print(f"  stall {nm.split('stalled_')[1][:-6]:30s} {s:.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
