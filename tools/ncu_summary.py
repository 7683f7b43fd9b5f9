"""Summarise an ncu report: per-kernel duration, DRAM bytes, hit rates and top stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [> profiles/rNN_summary.txt]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        print("=" * 100)
        print(name[:100])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:60s} {row[i]:>20s} {units[i]}")
        tot = sum(float(row[hdr.index(s)] or 0) for s in stalls) or 1.0
        top = sorted(((float(row[hdr.index(s)] or 0), s) for s in stalls), reverse=True)[:8]
        print("  stall samples (top 8, share of all samples):")
        for v, s in top:
            print(f"    {s.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * v / tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
