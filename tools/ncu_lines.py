"""Top source lines of an ncu report by warp-stall samples (cuda,sass source view)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kern:
    cmd += ["-k", kern]
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
cur, out = None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            samp, inst = float(r[4]), float(r[7])
        except ValueError:
            continue
        out.append((samp, inst, cur, r[0], r[1][:90]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print(f"total samples {ts:.0f}, warp instructions {ti:.3e}")
for o in sorted(out, reverse=True)[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{o[0] / ts * 100:5.1f}% samp {o[1] / ti * 100:5.1f}% inst  {o[2]}:{o[3]}  {o[4]}")
