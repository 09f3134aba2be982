"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

Usage: python scripts/launch_summary.py gpurun_out/launches.csv "<command line>" > profiles/rN_launches_summary.txt

Launches are split by ORDER into setup (everything before the first IPM kernel, k_ipm_mu:
factorization, inverses, accuracy guards, flattened-forest extraction) and step (the IPM
iterations), so the step-share of each kernel can be compared with bench.py's live
`fsolve_share_of_step`.
"""
import csv
import sys
from collections import defaultdict


def main(path, cmd):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
        val = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1.0}[unit]
        rows.append((int(r["ID"]), name, val * scale))
    first_ipm = min((i for i, n, _ in rows if n.startswith("k_ipm_")), default=0)
    setup, step = defaultdict(lambda: [0, 0.0]), defaultdict(lambda: [0, 0.0])
    for i, n, t in rows:
        d = setup if i < first_ipm else step
        d[n][0] += 1
        d[n][1] += t
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none: {cmd}")
    print("# (B200). Per-launch times are cold-cache and serialised: compare SHARES, not absolutes.")
    print(f"# {len(rows)} launches total; times in ns")
    for title, d in (("STEP kernels (IPM iterations: residuals, F-solves, PCG, recovery, step)", step),
                     ("SETUP kernels (ipm_factor_once: LDL^T, inverses, guards, forest extraction)", setup)):
        tot = sum(v[1] for v in d.values()) or 1.0
        print(f"\n## {title}: {sum(v[0] for v in d.values())} launches, {tot / 1e6:.3f} ms")
        print(f"{'kernel':40s} {'launches':>9s} {'sum_ns':>14s} {'avg_ns':>11s} {'share':>7s}")
        for k, (c, t) in sorted(d.items(), key=lambda kv: -kv[1][1]):
            print(f"{k:40s} {c:9d} {t:14.0f} {t / c:11.0f} {100 * t / tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
