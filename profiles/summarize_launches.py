"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X.csv):
    python profiles/summarize_launches.py gpurun_out/launches.csv "<header>" > profiles/<name>.txt
"""
import csv
import sys
from collections import OrderedDict


def main(path, header):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        ms = v / 1e6 if r.get("Metric Unit") == "ns" else v / 1e3 if r.get("Metric Unit") == "us" else v
        name = r["Kernel Name"].split("(")[0][:60]
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + ms)
    total = sum(t for _, t in agg.values())
    print(header)
    print(f"{'kernel':<60} {'launches':>8} {'total_ms':>10}  share")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:<60} {n:>8} {t:>10.3f} {100 * t / total:5.1f}%")
    print(f"{'total':<60} {sum(n for n, _ in agg.values()):>8} {total:>10.3f}")
    # headline = f64 rows: the 4th template argument (DF) is 0
    sgd = [(k, v) for k, v in agg.items()
           if "k_sgd_hogwild<" in k and k.split("<")[1].rstrip(">").split(",")[3].strip() == "0"]
    for k, (n, t) in sgd:
        print(f"\nheadline SGD kernel {k}: {n} launches, {t / n:.3f} ms per launch (cold-cache, serialised)")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
