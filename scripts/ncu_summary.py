"""Summarise an `ncu --set full` report (read with `ncu -i REP --page raw --csv`) per launch.

Usage: python scripts/ncu_summary.py REP.ncu-rep|RAW.csv "<capture command>" [config] [traffic.json]
Prints a per-launch table and, with a traffic.json path, records the DRAM bytes of one F-solve
(forward sweep + symmetric-root GEMV + backward sweep) for bench.py's roofline `traffic` key.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_read",
        "dram__bytes_write.sum": "dram_write", "dram__bytes_read.sum.pct_of_peak_sustained_elapsed": "dram_pct",
        "lts__t_sector_hit_rate.pct": "l2_hit_pct", "launch__registers_per_thread": "regs",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occ_pct",
        "smsp__issue_active.avg.per_cycle_active": "issue_active"}
SCALE = {"ns": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "Tbyte": 1e12}


def rows(rep):
    """rep: an .ncu-rep (read through ncu -i) or the CSV of `ncu -i REP --page raw --csv`."""
    if rep.endswith(".csv"):
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    head, units, data = r[0], r[1], r[2:]
    out = []
    for d in data:
        rec = {"kernel": d[head.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k, name in KEYS.items():
            if k not in head:
                continue
            i = head.index(k)
            v = float(d[i].replace(",", "")) if d[i] else float("nan")
            u = units[i]
            if name == "duration":
                v *= SCALE.get(u, 1.0)         # → µs
            elif name.startswith("dram_") and name != "dram_pct":
                v *= SCALE.get(u, 1.0)         # → bytes
            rec[name] = v
        out.append(rec)
    return out


def main():
    rep, cmd = sys.argv[1], sys.argv[2]
    cfg = sys.argv[3] if len(sys.argv) > 3 else "c1"
    recs = rows(rep)
    print(f"# ncu --set full --clock-control none: {cmd}")
    print(f"# {'kernel':30s} {'dur_us':>9s} {'DRAM rd GB':>10s} {'wr MB':>8s} {'DRAM %pk':>8s} {'GB/s':>8s} "
          f"{'L2 hit%':>7s} {'regs':>5s} {'occ%':>6s} {'issue':>6s}")
    for r in recs:
        gbs = (r["dram_read"] + r["dram_write"]) / (r["duration"] * 1e-6) / 1e9
        print(f"  {r['kernel']:30s} {r['duration']:9.1f} {r['dram_read'] / 1e9:10.4f} {r['dram_write'] / 1e6:8.2f} "
              f"{r['dram_pct']:8.1f} {gbs:8.0f} {r['l2_hit_pct']:7.1f} {r['regs']:5.0f} "
              f"{r['achieved_occ_pct']:6.1f} {r['issue_active']:6.2f}")
    if len(sys.argv) > 4:
        # one F-solve = one launch of each F-solve kernel (sweeps or flattened products, root GEMV)
        one, seen = [], set()
        for r in recs:
            k = r["kernel"].split("<")[0].strip()
            if k in ("k_trsv_fwd", "k_symroot_gemv", "k_trsv_bwd", "k_flat_rhs", "k_flat_fwd", "k_flat_bwd",
                     "k_flat_fwd_t", "k_flat_bwd_t") \
                    and k not in seen:
                seen.add(k)
                one.append(r)
        path = sys.argv[4]
        try:
            tj = json.load(open(path))
        except Exception:
            tj = {}
        prev = tj.get(cfg, {})
        w = [r for r in recs if r["kernel"].split("<")[0].strip() == "k_dense_symv"]
        if w:   # explicit W: one launch per PCG K_F product (kept beside the F-solve numbers)
            prev["dram_bytes_per_kf_W"] = w[0]["dram_read"] + w[0]["dram_write"]
            prev["kf_W_launch"] = {"kernel": w[0]["kernel"], "duration_us": w[0]["duration"],
                                   "dram_read_GB": w[0]["dram_read"] / 1e9, "dram_pct_of_peak": w[0]["dram_pct"],
                                   "source": f"ncu --set full --clock-control none: {cmd}"}
        if not one:
            tj[cfg] = prev
            json.dump(tj, open(path, "w"), indent=1)
            return
        prev.update({"dram_bytes_per_fsolve": sum(r["dram_read"] + r["dram_write"] for r in one),
                   "source": f"ncu --set full --clock-control none: {cmd}",
                   "launches": [{"kernel": r["kernel"], "duration_us": r["duration"],
                                 "dram_read_GB": r["dram_read"] / 1e9, "dram_write_MB": r["dram_write"] / 1e6,
                                 "dram_pct_of_peak": r["dram_pct"]} for r in one]})
        tj[cfg] = prev
        json.dump(tj, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
