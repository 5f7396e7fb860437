"""Build variants of the CUDA library for A/B timing: ab/<name>.so with extra nvcc flags.

    python tools/build_ab.py minb3 -DFSB_STO_MINB=3
    FSB_LIB=ab/minb3.so python tools/ab_sto.py      (on the GPU box)
"""
import os
import subprocess
import sys
import concurrent.futures as cf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_02219_b200 import _build as B  # noqa: E402


def build(name, extra):
    out_dir = os.path.join(ROOT, "ab", name)
    os.makedirs(out_dir, exist_ok=True)
    nv = B.nvcc()

    def one(src):
        obj = os.path.join(out_dir, src.replace(".cu", ".o"))
        subprocess.run([nv, *B.flags(), *extra, "-c", os.path.join(B.CSRC, src), "-o", obj],
                       check=True)
        return obj

    with cf.ThreadPoolExecutor(len(B.SOURCES)) as ex:
        objs = list(ex.map(one, B.SOURCES))
    lib = os.path.join(ROOT, "ab", name + ".so")
    subprocess.run([nv, *B.ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"], check=True)
    for o in objs:
        os.remove(o)
    os.rmdir(out_dir)
    return lib


if __name__ == "__main__":
    print(build(sys.argv[1], sys.argv[2:]))
