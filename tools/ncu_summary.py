"""Summarise one kernel of an ncu --set full report (ncu -i ... --page raw --csv) into the
numbers the roofline uses: duration, DRAM bytes and throughput, SM/tensor pipe use, stalls."""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "gpc__cycles_elapsed.max",
]


def main(rep, kernel_filter=""):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        if kernel_filter not in d.get("Kernel Name", ""):
            continue
        print("kernel:", d.get("Kernel Name"))
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k} = {row[i]} {units[i]}")
        rd = wr = None
        for k, v in d.items():
            pass
        try:
            i_r, i_w = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(row[i_r].replace(",", "")) * scale[units[i_r]]
            wr = float(row[i_w].replace(",", "")) * scale[units[i_w]]
            print(f"  dram bytes (read + write) per launch = {rd + wr:.0f}")
        except (ValueError, KeyError):
            pass


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
