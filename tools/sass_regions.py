"""Split an ncu SASS source dump into regions at branch targets and report
executed (thread) instructions per region, to see where a kernel spends issue slots."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x.replace(',', ''))
    except ValueError:
        return 0.0


tot = sum(num(d["Thread Instructions Executed"]) for d in data)
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 40
acc, acc_w, samples, first = 0.0, 0.0, 0.0, None
for i, d in enumerate(data):
    if first is None:
        first = d
    acc += num(d["Thread Instructions Executed"])
    acc_w += num(d["Instructions Executed"])
    samples += num(d["Warp Stall Sampling (All Samples)"])
    if (i + 1) % chunk == 0 or i == len(data) - 1:
        if acc / tot > 0.005:
            ops = {}
            for dd in data[i + 1 - chunk if i + 1 >= chunk else 0:i + 1]:
                p = dd["Source"].split()
                if p:
                    op = (p[1] if p[0].startswith("@") and len(p) > 1 else p[0]).split(".")[0]
                    ops[op] = ops.get(op, 0) + 1
            key = ",".join(k for k, _ in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
            eff = acc / max(acc_w, 1) / 32
            print(f"{first['Address'][-5:]} thr-instr {acc/tot:6.3f} eff {eff:4.2f} "
                  f"stall {samples:7.0f}  {key}")
        acc, acc_w, samples, first = 0.0, 0.0, 0.0, None
