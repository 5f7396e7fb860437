"""DRAM bytes and GPU time of the tree-build kernels (the build is
HBM-bound).  Two steps, on the GPU box:

    ncu --nvtx --nvtx-include "warm_build/" --metrics \
        dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --csv --log-file gpurun_out/build_ncu.csv python tools/profile_build.py run
    python tools/profile_build.py summarize gpurun_out/build_ncu.csv profiles/r02_build.json

`run` builds the C4 d = 4 tree from device-resident inputs once (cold) and once
more inside the NVTX range `warm_build` (the measured one).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run():
    import ctypes as C
    import torch
    import bench
    from paper_2506_02219_b200 import _device as dev, _lib
    src, _, _ = bench.workload()
    L = _lib.lib()
    pos, ms, w = (dev.to_device(a) for a in (src.positions, src.masses, src.weights))
    sp = C.c_void_p(dev.stream_ptr())

    def build():
        h = C.c_void_p()
        _lib.check(L.fsb_build_tree(C.c_void_p(dev.ptr(pos)), C.c_void_p(dev.ptr(ms)),
                                    C.c_void_p(dev.ptr(w)), len(src), 1, 4, 32, C.byref(h), sp))
        torch.cuda.synchronize()
        L.fsb_tree_free(h)

    build()
    with torch.cuda.nvtx.range("warm_build"):
        build()
    torch.cuda.synchronize()


def summarize(csv_path, out_path):
    rows = list(csv.reader(open(csv_path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    col = {k: h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID")}
    per = {}
    for r in rows[hdr + 1:]:
        if len(r) < len(h):
            continue
        k = per.setdefault(r[col["ID"]], {"name": r[col["Kernel Name"]]})
        k[r[col["Metric Name"]]] = float(r[col["Metric Value"]].replace(",", ""))
    rd = sum(k.get("dram__bytes_read.sum", 0.0) for k in per.values())
    wr = sum(k.get("dram__bytes_write.sum", 0.0) for k in per.values())
    t = sum(k.get("gpu__time_duration.sum", 0.0) for k in per.values())
    unit_t = "ns"
    names = sorted({k["name"].split("(")[0][:60] for k in per.values()})
    side = {"dram_bytes_total": rd + wr, "dram_read": rd, "dram_write": wr,
            "gpu_time_ms": t / 1e6 if unit_t == "ns" else t, "kernels": len(per),
            "kernel_names": names,
            "how": "ncu --nvtx --nvtx-include warm_build/ (serialised, cold caches per launch)"}
    json.dump(side, open(out_path, "w"), indent=1)
    print(json.dumps(side, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        summarize(sys.argv[2], sys.argv[3])
