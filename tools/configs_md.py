"""Format tools/configs.py JSON lines as profiles/rNN_configs.md.

    python tools/configs_md.py gpurun_out/configs.jsonl > profiles/r01_configs.md
"""
import json
import sys


def fmt(x, f="{:.3f}"):
    return "n/a" if x is None else f.format(x)


rows = [json.loads(line) for line in open(sys.argv[1]) if line.strip()]
print(f"# {sys.argv[2] if len(sys.argv) > 2 else 'Round 1'} -- secondary configs on one B200 (tools/configs.py)\n")
print("S=1 stochastic (FP32, paper_ratio, seed 1, d=4) with the reference's per-query RNG streams and with")
print("the paper's warp-shared streams, vs the GPU deterministic BH (FP32, load-balanced, d=2) swept over")
print("beta and log-log interpolated to each S=1 error (PAPER.md:312). Times are device-resident steps")
print("(CUDA events, tree prebuilt; best of 3 trials, SM clocks sampled: no throttling). Ground truth:")
print("GPU brute force, FP32 terms / FP64 accumulation.")
print("C4 (the headline) is in bench.py.\n")
print("| config | workload | queries | error metric | per-query: ms / error / speed-up | "
      "warp-shared: ms / error / speed-up | matched BH ms |")
print("|---|---|---:|---|---:|---:|---:|")
for r in rows:
    w = r["warp_streams"]
    sp = r["speedup_at_matched_error"]
    spw = w["speedup_at_matched_error"]
    print(f"| {r['config']} | {r['workload']} | {r['queries']:,} | {r['error_metric']} | "
          f"{r['s1_ms']:.3f} / {r['s1_err']:.2e} / {fmt(sp, '{:.2f}x')} | "
          f"{w['s1_ms']:.3f} / {w['s1_err']:.2e} / {fmt(spw, '{:.2f}x')} | "
          f"{fmt(r['matched_bh_ms'])} |")
print("\nBH sweeps (beta: ms, error):\n")
for r in rows:
    pts = ", ".join(f"{p['beta']}: {p['ms']:.2f} ms / {p['err']:.2e}" for p in r["bh_sweep"])
    extra = f"; flagged fraction {r['flagged_fraction']:.3f}" if "flagged_fraction" in r else ""
    print(f"* {r['config']}: {pts}{extra}")
