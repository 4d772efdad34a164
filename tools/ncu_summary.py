"""Summarise ncu --set full reports (.ncu-rep) into a compact JSON + markdown table.

usage: python tools/ncu_summary.py OUT_PREFIX REP [REP ...]
Writes OUT_PREFIX.json and OUT_PREFIX.md (commit them under profiles/).
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "duration_us": ("gpu__time_duration.sum", {"ms": 1e3, "us": 1.0, "ns": 1e-3, "msecond": 1e3,
                                                "usecond": 1.0, "nsecond": 1e-3}),
    "dram_read_GB": ("dram__bytes_read.sum", {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}),
    "dram_write_GB": ("dram__bytes_write.sum", {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}),
    "dram_read_pct": ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", None),
    "dram_write_pct": ("dram__bytes_write.sum.pct_of_peak_sustained_elapsed", None),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", None),
    "l2_read_hit_pct": ("lts__t_sector_op_read_hit_rate.pct", None),
    "l1_ld_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", None),
    "l1_ld_requests": ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", None),
    "l1_ld_wavefronts": ("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum", None),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", None),
    "lts_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "l1_throughput_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "registers": ("launch__registers_per_thread", None),
    "grid": ("launch__grid_size", None),
    "occ_limit_regs": ("launch__occupancy_limit_registers", None),
    "occ_limit_smem": ("launch__occupancy_limit_shared_mem", None),
    "cycles_per_issue": ("smsp__average_warp_latency_per_inst_issued.ratio", None),
    "stall_long_scoreboard": ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", None),
    "stall_wait": ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", None),
    "stall_lg_throttle": ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", None),
    "stall_mio_throttle": ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", None),
    "stall_short_scoreboard": ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", None),
    "inst_executed": ("smsp__inst_executed.sum", None),
    "local_spill_req": ("l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum", None),
}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {"report": os.path.basename(rep), "kernel": d.get("Kernel Name", "")[:80]}
        for k, (m, conv) in METRICS.items():
            if m not in d or d[m] == "":
                continue
            v = float(d[m].replace(",", ""))
            if conv:
                u = units[hdr.index(m)]
                v *= conv.get(u, 1.0)
            e[k] = round(v, 4)
        if e.get("l1_ld_requests"):
            e["l1_sectors_per_request"] = round(e["l1_ld_sectors"] / e["l1_ld_requests"], 3)
        if "dram_read_GB" in e and "dram_write_GB" in e:
            e["dram_traffic_GB"] = round(e["dram_read_GB"] + e["dram_write_GB"], 4)
        res.append(e)
    return res


def main():
    prefix, reps = sys.argv[1], sys.argv[2:]
    allr = []
    for r in reps:
        allr += summarise(r)
    json.dump(allr, open(prefix + ".json", "w"), indent=1)
    keys = ["report", "kernel", "duration_us", "dram_traffic_GB", "dram_read_pct", "l2_hit_pct",
            "l2_read_hit_pct", "l1_hit_pct", "l1_sectors_per_request", "lts_throughput_pct",
            "warps_active_pct", "registers", "cycles_per_issue", "stall_long_scoreboard"]
    with open(prefix + ".md", "w") as f:
        f.write("| " + " | ".join(keys) + " |\n|" + "---|" * len(keys) + "\n")
        for e in allr:
            f.write("| " + " | ".join(str(e.get(k, "")) for k in keys) + " |\n")
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    main()
