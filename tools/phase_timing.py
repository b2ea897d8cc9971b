"""Per-CTA phase timing of one SpMM launch using an instrumented build (-DSTEN_TIMING).

    python tools/phase_timing.py --M 768 --K 770 --N 1024 --n 1 --m 10 --tile 3 --split 4
"""
import argparse, ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
DBG = os.path.join(ROOT, "paper_2304_07613_b200", "libsten_timing.so")


def lib_path(exp, tag=""):
    return DBG.replace(".so", "%s%s.so" % ("_exp%d" % exp if exp else "", "_" + tag if tag else ""))


def build(exp=0, defs="", tag=""):
    from paper_2304_07613_b200 import build as b
    extra = ["-D" + d for d in defs.split(",") if d]
    cmd = [b.NVCC] + b.ARCH + b.FLAGS + ["-DSTEN_TIMING", "-DSTEN_TC_EXP=%d" % exp] + extra + [
        "-I", b.INCLUDE, "-I", b.CSRC, "-o", lib_path(exp, tag)] + sorted(
        os.path.join(b.CSRC, f) for f in os.listdir(b.CSRC) if f.endswith(".cu"))
    subprocess.check_call(cmd)


def main():
    p = argparse.ArgumentParser()
    for k, v in dict(M=768, K=3072, N=1024, n=2, m=4, g=4, tile=0, split=0).items():
        p.add_argument("--" + k, type=int, default=v)
    p.add_argument("--build", action="store_true")
    p.add_argument("--exp", type=int, default=0, help="STEN_TC_EXP experiment build (timing only)")
    p.add_argument("--defs", default="", help="extra -D defines for --build, comma separated")
    p.add_argument("--timeline", default="", help="print CTA 0's per-slab event timeline (legend)")
    p.add_argument("--tag", default="", help="library tag for --defs builds")
    p.add_argument("--algo", type=int, default=1)
    p.add_argument("--dtype", default="f32")
    p.add_argument("--wait_names", default="prod empty wait,mma full wait,mma aready wait,gather full wait,"
                   "gather afree wait,gather work,mma loop total,gather loop total")
    p.add_argument("--names", default="start,setup+issue,slab0 ready,main loop done,tile parked,reduced")
    a = p.parse_args()
    if a.build:
        build(a.exp, a.defs, a.tag)
        return
    os.environ["STEN_LIB_PATH"] = lib_path(a.exp, a.tag)
    import numpy as np
    import torch
    from paper_2304_07613_b200 import sten
    lib = sten.load()
    lib.sten_debug_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
    dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    W = (torch.randn(a.M, a.K, device="cuda") * 0.02).to(dt)
    B = torch.randn(a.K, a.N, device="cuda").to(dt)
    v, i = sten.sparsify_grouped_nm(W, a.n, a.m, a.g)
    plan = sten.make_plan(a.algo, max(1, a.split), a.tile) if a.tile else None
    lib.sten_debug_waits.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    for _ in range(3):
        lib.sten_debug_waits(None, 0, 1)
        C = sten.spmm_grouped_nm(v, i, B, a.n, a.m, a.g, plan=plan)
    torch.cuda.synchronize()
    if a.timeline:
        tl = np.zeros((256, 8), dtype=np.int64)
        lib.sten_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.sten_debug_timeline(tl.ctypes.data, 0)
        tl2 = np.zeros((256, 8), dtype=np.int64)
        lib.sten_debug_timeline(tl2.ctypes.data, 1)
        t0 = tl[0, 0]
        print("timeline of CTA 0 (cycles from slab 0 issue): " + a.timeline)
        for k in range(256):
            if tl[k, 0] == 0:
                break
            print("  slab %3d " % k + " ".join("%8d" % (v - t0 if v else -1) for v in tl[k, :8]))
        print("gather warp 4 units (cycles from slab 0 issue): afree-done, addr-done, sttm-issued, wait-st-done")
        for k in range(256):
            if tl2[k, 0] == 0:
                continue
            print("  unit %3d " % k + " ".join("%8d" % (v - t0 if v else -1) for v in tl2[k, :4]))
            if k > 60:
                break
    wb = np.zeros((16384, 8), dtype=np.uint64)
    lib.sten_debug_waits(wb.ctypes.data, 16384, 0)
    wnames = a.wait_names.split(",")
    wrows = wb[wb.sum(axis=1) > 0].astype(np.float64)
    if len(wrows):
        print("accumulated cycles per CTA (mean):")
        for k in range(8):
            if wrows[:, k].any():
                print("  %-22s %10.0f" % (wnames[k] if k < len(wnames) else str(k), wrows[:, k].mean()))
    buf = np.zeros((16384, 8), dtype=np.uint64)
    lib.sten_debug_timing(buf.ctypes.data, 16384)
    rows = buf[buf[:, 0] > 0].astype(np.int64)
    t0 = rows[:, 0].min()
    names = a.names.split(",")
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
