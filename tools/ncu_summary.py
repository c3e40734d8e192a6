"""Summarise the ncu evidence of one round into profiles/ (run here, on the CPU).

    python tools/ncu_summary.py r01 [workload]

Reads gpurun_out/prof_<r>/{launches.csv, featurize.ncu-rep, predict.ncu-rep}
(tools/profile_round.sh) and writes
  profiles/ncu_<r>_<workload>.md      human summary (launch shares, key counters)
  profiles/ncu_traffic.json           per-workload numbers bench.py reads for its
                                      roofline object (dram bytes, instructions per launch)
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
    "sm__inst_executed.sum.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
         "s": 1.0, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    h, units = rows[0], rows[1]
    m = {}
    for vals in rows[2:]:  # one row per captured launch: additive counters are summed
        for k, u, v in zip(h, units, vals):
            if k in KEYS:
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                x = x * SCALE.get(u, 1.0) if u in SCALE else x
                additive = k.endswith(".sum") and "per_" not in k
                m[k] = m.get(k, 0.0) + x if additive else x
                m[k + ".unit"] = u
        m["kernel"] = next((v for k, v in zip(h, vals) if k == "Kernel Name"), "")
    m["launches_captured"] = len(rows) - 2
    return m


def launches(path):
    per = defaultdict(lambda: [0, 0.0])
    if not os.path.exists(path):
        return per
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        m = re.search(r"(\w+)\s*(<[^()]*>)?\s*\(", r[ki].replace("(anonymous namespace)", ""))
        name = m.group(1) if m else r[ki][:60]
        val = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        per[name][0] += 1
        per[name][1] += val
    return per


def main():
    r = sys.argv[1] if len(sys.argv) > 1 else "r01"
    w = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
    d = os.path.join(ROOT, "gpurun_out", f"prof_{r}_{w}")
    if not os.path.isdir(d):
        d = os.path.join(ROOT, "gpurun_out", f"prof_{r}")
    lines = [f"# ncu evidence, round {r}, workload {w}", "",
             "Captured with tools/profile_round.sh on one B200 (`--clock-control none`).",
             "Launch times are cold-cache and serialised (compare shares, not absolutes).", ""]
    per = launches(os.path.join(d, "launches.csv"))
    tot = sum(v[1] for v in per.values()) or 1.0
    lines += ["## Launch list (all kernels of `bench.py --steps 2 --warmup 3`)", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {n} | {t*1e3:.3f} | {t/tot:.1%} |")
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    tw = traffic[w] = {}  # one capture per workload: no keys left over from an earlier one
    for tag in ("featurize", "predict"):
        rep = os.path.join(d, f"{tag}.ncu-rep")
        if not os.path.exists(rep):
            continue
        m = raw_metrics(rep)
        nl = int(m.get("launches_captured", 1))
        lines += ["", f"## `ncu --set full`: {tag} ({m.get('kernel', '')[:90]})",
                  "" if nl == 1 else f"\n{nl} launches captured (one step); additive counters summed.", "",
                  "| counter | value |",
                  "|---|---|"]
        for k in KEYS:
            if k in m:
                lines.append(f"| {k} | {m[k]:.6g} |")
        dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        kn = m.get("kernel", "")
        name = "attn_schedule_cross" if "attn_schedule" in kn else (
            "uniform_prepass" if "uniform_prepass" in kn else (
                "featurize_splitk_cross" if "splitk" in kn else (
                    "featurize_uniform_cross" if "uniform" in kn else None)))
        if tag == "predict":
            pk = "predict_tcgen05_fused" if "fused" in kn else "predict_tcgen05"
            for p in ("fp16", "bf16"):
                tw[f"{pk}_{p}_dram_bytes"] = dram
        elif name:
            tw[f"{name}_dram_bytes"] = dram
            tw[f"{name}_inst_executed"] = m.get("smsp__inst_executed.sum")
            tw.pop("featurize_inst_executed", None)
            tw.pop("featurize_attention_cross_dram_bytes", None)
        tw[f"{tag}_ncu_duration_s"] = m.get("gpu__time_duration.sum")
    tw["source"] = f"profiles/ncu_{r}_{w}.md"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"ncu_{r}_{w}.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
