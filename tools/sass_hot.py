"""Summarise an ncu --page source --csv (SASS) dump: top stall lines and opcode mix."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x.replace(',', ''))
    except ValueError:
        return 0.0


tot_s = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
tot_i = sum(num(d["Instructions Executed"]) for d in data)
tot_t = sum(num(d["Thread Instructions Executed"]) for d in data)
print(f"samples {tot_s:.0f} warp-instr {tot_i:.3e} thread-instr {tot_t:.3e} simt-eff {tot_t/max(tot_i,1)/32:.2f}")
ops = collections.Counter()
opss = collections.Counter()
for d in data:
    parts = d["Source"].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    op = op.split(".")[0]
    ops[op] += num(d["Instructions Executed"])
    opss[op] += num(d["Warp Stall Sampling (All Samples)"])
print("opcode mix (warp-instr share, stall-sample share):")
for op, c in ops.most_common(25):
    print(f"  {op:10s} {c/tot_i:6.3f} {opss[op]/max(tot_s,1):6.3f}")
k = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print("top lines by stall samples:")
stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
for d in sorted(data, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:k]:
    top = sorted(((num(d[c]), c) for c in stalls), reverse=True)[:2]
    print(f"  {d['Address']:>6} {num(d['Warp Stall Sampling (All Samples)'])/tot_s:6.3f} "
          f"thr={num(d['Avg. Threads Executed']):5.1f} {d['Source'][:58]:58s} "
          f"{top[0][1]}:{top[0][0]:.0f} {top[1][1]}:{top[1][0]:.0f}")
