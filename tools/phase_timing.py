"""Per-CTA phase timing of one SpMM launch using an instrumented build (-DSTEN_TIMING).

    python tools/phase_timing.py --M 768 --K 770 --N 1024 --n 1 --m 10 --tile 3 --split 4
"""
import argparse, ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
DBG = os.path.join(ROOT, "paper_2304_07613_b200", "libsten_timing.so")


def build():
    from paper_2304_07613_b200 import build as b
    cmd = [b.NVCC] + b.ARCH + b.FLAGS + ["-DSTEN_TIMING", "-I", b.INCLUDE, "-I", b.CSRC, "-o", DBG,
                                         os.path.join(b.CSRC, "sten_api.cu")]
    subprocess.check_call(cmd)


def main():
    p = argparse.ArgumentParser()
    for k, v in dict(M=768, K=3072, N=1024, n=2, m=4, g=4, tile=0, split=0).items():
        p.add_argument("--" + k, type=int, default=v)
    p.add_argument("--build", action="store_true")
    a = p.parse_args()
    if a.build:
        build()
        return
    os.environ["STEN_LIB_PATH"] = DBG
    import numpy as np
    import torch
    from paper_2304_07613_b200 import sten
    lib = sten.load()
    lib.sten_debug_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
    W = torch.randn(a.M, a.K, device="cuda") * 0.02
    B = torch.randn(a.K, a.N, device="cuda")
    v, i = sten.sparsify_grouped_nm(W, a.n, a.m, a.g)
    plan = sten.make_plan(1, a.split, a.tile) if a.tile else None
    for _ in range(3):
        C = sten.spmm_grouped_nm(v, i, B, a.n, a.m, a.g, plan=plan)
    torch.cuda.synchronize()
    buf = np.zeros((16384, 8), dtype=np.uint64)
    lib.sten_debug_timing(buf.ctypes.data, 16384)
    rows = buf[buf[:, 0] > 0].astype(np.int64)
    t0 = rows[:, 0].min()
    names = ["start", "setup+issue", "slab0 ready", "main loop done", "tile parked", "reduced"]
    print("ctas", len(rows))
    print("start spread (us): min 0 max %.2f" % ((rows[:, 0].max() - t0) / 1e3))
    for k in range(1, 6):
        ok = rows[:, k] > 0
        if not ok.any():
            continue
        d = (rows[ok, k] - rows[ok, k - 1]) / 1e3 if (rows[ok, k - 1] > 0).all() else None
        if d is not None:
            print("%-16s mean %.2f us  max %.2f us" % (names[k], d.mean(), d.max()))
    last = rows[:, 1:6].max(axis=1)
    print("cta end (us from first start): mean %.2f max %.2f" % (((last - t0) / 1e3).mean(), (last.max() - t0) / 1e3))


if __name__ == "__main__":
    main()
