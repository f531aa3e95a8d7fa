"""Extract the judged counters of one kernel from an ncu --set full report into
profiles/traffic.json (keyed by workload), which bench.py reads for `roofline.traffic`
and `roofline.ncu`.

  python scripts/ncu_extract.py <report.ncu-rep> <kernel-regex> <workload> [prefix]
"""
import csv
import io
import json
import os
import subprocess
import sys

WANT = {
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__time_duration.sum": "duration_ns",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "avg_active_threads_per_warp",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__thread_inst_executed.sum": "thread_instructions",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_active_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_rate_pct",
}


def main():
    rep, kern, workload = sys.argv[1], sys.argv[2], sys.argv[3]
    prefix = sys.argv[4] if len(sys.argv) > 4 else "k_step"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name", f"regex:{kern}"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    got = {}
    for i, h in enumerate(hdr):
        if h in WANT:
            v = vals[i].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[i]
            if u == "Kbyte":
                x *= 1e3
            elif u == "Mbyte":
                x *= 1e6
            elif u == "Gbyte":
                x *= 1e9
            elif u in ("usecond", "us"):
                x *= 1e3
            elif u in ("msecond", "ms"):
                x *= 1e6
            got[WANT[h]] = x
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    ent = data.setdefault(workload, {})
    if "dram_read_bytes" in got and "dram_write_bytes" in got:
        ent[f"{prefix}_dram_bytes"] = got["dram_read_bytes"] + got["dram_write_bytes"]
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import source_sha  # the revision this capture measured (bench.py checks it)
    ent[f"{prefix}_ncu"] = dict(got, report=os.path.basename(rep), source_sha=source_sha())
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps({workload: ent}, indent=1))


if __name__ == "__main__":
    main()
