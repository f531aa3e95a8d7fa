"""Markdown summary of one scripts/gpu_check_r02.sh run (bench lines, kernel launch list, ncu
counters of k_step / k_lp3 / k_scan / k_scatter), for profiles/SUMMARY_*.md.
  python scripts/summarize_run.py <tag> [gpurun_out]"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

tag = sys.argv[1]
d = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"


def line(f):
    try:
        return json.loads(open(os.path.join(d, f)).read().strip().splitlines()[-1])
    except Exception:
        return None


print(f"### Bench lines ({tag})\n")
print("| workload | ms/step | agent-updates/s | roofline frac (SURVEY work) | executed frac | peak (measured) | "
      "k_step+k_lp3 / scan / scatter ms | e2e ms/frame | kernels/step |")
print("|---|---|---|---|---|---|---|---|---|")
for f in (f"bench_{tag}.json", f"bench100k_{tag}.json", f"benchdense_{tag}.json"):
    b = line(f)
    if not b:
        continue
    r = b["roofline"]
    st = r["stage_ms"]
    print(f"| {b['config']['workload']} | {b['ms_per_step']:.4f} | {b['value']:.3e} | {r['frac']:.3f} | "
          f"{r['frac_executed']:.3f} | {r['peak']:.2f} T lane-op/s | {st['k_step+k_lp3']:.4f} / {st['k_scan']:.4f} / "
          f"{st['k_scatter']:.4f} | {b['e2e']['ms_per_step']:.4f} | {b['launch_info']['kernels_per_step']} |")
ref = line(f"ref_{tag}.json")
if ref:
    print(f"\nReference arm (fp64 oracle): {ref['value']:.3e} agent-updates/s, {ref['steps']} full steps of "
          f"{ref['config']['n_agents']} agents, {ref['cpu_baseline']['cores']} cores "
          f"({ref['cpu_baseline']['cpu_model']}).")
b = line(f"bench_{tag}.json")
if b and b.get("cpu_baseline"):
    cb = b["cpu_baseline"]
    print(f"cpu_baseline: {cb['value']:.3e} agent-updates/s on {cb['cores']} cores; single thread "
          f"{cb['single_thread']['value']:.3e}; C0/C1 full runs: "
          + ", ".join(f"{k} {v['ms_per_frame']:.2f} ms/frame" for k, v in cb.get('configs_full_runs', {}).items()))
if b and b.get("clocks"):
    print(f"clocks during the timed region: {b['clocks']}")

for lf, name in ((f"launches_{tag}.csv", "1M"), (f"launches100k_{tag}.csv", "100k")):
    p = os.path.join(d, lf)
    if not os.path.exists(p):
        continue
    rows = [r for r in csv.reader(open(p)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    dd = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            dd[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
    # the step's own kernels: every non-debug k_step / k_lp3 instantiation, the scan, the scatter
    main = [k for k in dd if (k.startswith("void orca::k_step<0,") or k.startswith("void orca::k_lp3<0"))] + \
        ["orca::k_scan", "orca::k_scatter"]
    med = {k: sorted(v)[len(v) // 2] / 1000 for k, v in dd.items()}
    tot = sum(med.get(k, 0) for k in main)
    print(f"\n### ncu launch list, {name} (cold cache, serialised; median per launch)\n")
    print("| kernel | µs | share of the step |")
    print("|---|---|---|")
    for k in main:
        if k in med:
            print(f"| {k.split('::')[-1]} | {med[k]:.1f} | {100 * med[k] / tot:.1f} % |")


def ncu_details(rep, regex):
    p = os.path.join(d, rep)
    if not os.path.exists(p):
        return {}
    out = subprocess.run(["ncu", "-i", p, "--page", "details", "--csv", "-k", f"regex:{regex}"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        return {}
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    res = collections.OrderedDict()
    for r in rows[1:]:
        res.setdefault(r[ki].split("(")[0], {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    return res


want = ["Duration", "Issued Instructions", "Issue Slots Busy", "Avg. Active Threads Per Warp", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "L1/TEX Hit Rate", "DRAM Throughput", "Memory Throughput"]
for rep, rx, name in ((f"prof_kstep_{tag}.ncu-rep", "k_step|k_lp3", "1M"), (f"prof_kstep100k_{tag}.ncu-rep", "k_step", "100k"),
                      (f"prof_bin_{tag}.ncu-rep", "k_scan|k_scatter", "binning")):
    det = ncu_details(rep, rx)
    for k, m in det.items():
        print(f"\n**{k}** ({name}, ncu --set full): " + "; ".join(f"{w} {m[w]}" for w in want if w in m))
