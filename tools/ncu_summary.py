#!/usr/bin/env python
"""Extracts the judged numbers from an .ncu-rep (read here, no GPU needed):
   python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_verify   ->  *_metrics.csv, *_opmix.csv
"""
import collections
import csv
import re
import subprocess
import sys

KEEP = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "dram__bytes_write.sum.per_second",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sass__inst_executed_local_loads",
        "sass__inst_executed_local_stores", "sass__inst_executed_shared_loads", "sass__inst_executed_shared_stores",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__cycles_elapsed.max",
        "l1tex__t_sector_pipe_lsu_mem_local_op_ld_hit_rate.pct"]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    with open(out + "_metrics.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "metric", "unit", "value"])
        for vals in rows[2:]:
            name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
            for h, u, v in zip(hdr, units, vals):
                if h in KEEP or h.startswith("smsp__average_warps_issue_stalled"):
                    w.writerow([name.split("(")[0].replace("void ", "")[:60], h, u, v])
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    hdr = rows[1]
    ia, isrc, isamp, iex = (hdr.index(k) for k in ("Address", "Source", "# Samples", "Instructions Executed"))
    ex, sm = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= iex or not r[ia].startswith("0x"):
            continue
        m = re.match(r"(@!?U?P\d+\s+)?([A-Z0-9_.]+)", r[isrc].strip())
        op = m.group(2) if m else "?"
        if op.startswith("IMAD"):
            op = ("IMAD.WIDE" if "WIDE" in op else "IMAD.HI" if ".HI" in op else "IMAD.MOV" if "MOV" in op
                  else "IMAD.X" if ".X" in op else "IMAD")
        else:
            op = op.split(".")[0]
        ex[op] += int(r[iex])
        sm[op] += int(r[isamp])
    te, ts = sum(ex.values()), sum(sm.values())
    with open(out + "_opmix.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["opcode", "warp_instructions_executed", "executed_pct", "stall_samples_pct"])
        for op, e in ex.most_common(30):
            w.writerow([op, e, f"{100 * e / te:.2f}", f"{100 * sm[op] / ts:.2f}"])
    print("wrote", out + "_metrics.csv", out + "_opmix.csv")


if __name__ == "__main__":
    main()
