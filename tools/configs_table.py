"""Format gpurun_out/cfg_*.json (tools/configs_run.sh) as the profiles/r1_configs.txt table."""
import json
import os

print(f"{'cfg':<5}{'value':>10}{'ms/ep':>8}{'HBM frac':>9}{'e2e':>10}{'DF rows':>10}"
      f"{'cpu(same idx)':>17}{'ref arm':>10}{'kNN exact s':>12}{'recall':>7}{'SM MHz':>7}  workload")
for c in ["A", "B", "C8", "C"]:
    f = f"gpurun_out/cfg_{c}.json"
    if not os.path.exists(f) or not os.path.getsize(f):
        continue
    d = json.load(open(f))
    r = json.load(open(f"gpurun_out/cfg_{c}_ref.json")) if os.path.getsize(f"gpurun_out/cfg_{c}_ref.json") else {}
    cpu = d.get("cpu_baseline") or {}
    idx = d["config"].get("index", {})
    print(f"{c:<5}{d['value']:>10.3g}{d['ms_per_step']:>8.3f}{d['roofline']['frac']:>9.3f}"
          f"{d['e2e']['value']:>10.3g}{d['double_float_rows']['value']:>10.3g}"
          f"{cpu.get('value', float('nan')):>13.3g} x{cpu.get('cores', '-'):<2}{r.get('value', float('nan')):>10.3g}"
          f"{idx.get('build_knn_s', float('nan')):>12.2f}{idx['knn_recall_at_15']['value']:>7.3f}"
          f"{d['clocks']['sm_mhz']:>7.0f}  {d['config']['workload']}")
