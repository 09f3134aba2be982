"""Top CUDA source lines by warp-stall samples of one kernel in an ncu report (needs -lineinfo)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_ins = hdr.index("Instructions Executed")
out = []
for r in rows:
    if len(r) == len(hdr) and r[0] not in ("", "Line No"):
        try:
            out.append((float(r[i_s] or 0), float(r[i_ins] or 0), r[0], r[1].strip()))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
toti = sum(o[1] for o in out) or 1
print(f"{kern}: {tot:.0f} stall samples, {toti:.3g} warp instructions")
for s, ins, ln, src in sorted(out, reverse=True)[:n]:
    print(f"  {100 * s / tot:5.1f}% stalls {100 * ins / toti:5.1f}% inst  L{ln}: {src[:100]}")
