"""Summarise an .ncu-rep: key throughput/occupancy metrics and top stall reasons per kernel."""
import csv, subprocess, sys, io, re

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]

def main(rep):
    hdr, units, rows = raw(rep)
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        print("==", name[:110])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {k} = {r[i]} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", h)
            if m and not h.endswith("not_issued") and r[i] not in ("", "0"):
                stalls.append((float(r[i].replace(",", "")), m.group(1)))
        tot = sum(v for v, _ in stalls) or 1
        print("   stalls:", ", ".join(f"{n} {v / tot:.0%}" for v, n in sorted(stalls, reverse=True)[:8]))

if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
