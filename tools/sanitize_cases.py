"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): K1 sparsify (+ grouped), K2 densify, K3 SIMT SpMM (tiles 1-7, split-K cluster and the
grouped workspace path, fused epilogue with residual), K4 mma.sync, K5 tcgen05, K6 2:4 sparse
tcgen05 (+ pack), the chunked n:m:g conversion (greedy / exchange) and SpMM, SDDMM, mask check.
Checks each result against the oracle on the side (a sanitizer-perturbed run must still be right)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synthetic  # noqa: E402
from paper_2304_07613_b200 import sten  # noqa: E402
from test_gpu_parity import dev, rel_err  # noqa: E402

which = set(sys.argv[1].split(",")) if len(sys.argv) > 1 else None


def on(name):
    return which is None or name in which


def ok(name, cond):
    print("CASE %s %s" % (name, "ok" if cond else "FAIL"), flush=True)


n, m, g, M, K, N = 2, 4, 4, 120, 256, 136
W = synthetic.weights(M, K, seed=1)
B = synthetic.activations(K, N, seed=2)
v_ref, i_ref = oracle.sparsify(W, n, m, g)
C_ref, Bd = oracle.spmm(v_ref, i_ref, B, n, m, g)
Wd, Bdv = dev(W, "f32"), dev(B, "f32")
if on("k1"):
    v, i = sten.sparsify_grouped_nm(Wd, n, m, g)
    torch.cuda.synchronize()
    ok("k1 sparsify", np.array_equal(i.cpu().numpy(), i_ref))
    vals = torch.empty_like(v)
    idx = torch.empty_like(i)
    sten.sparsify_grouped_nm_batched([(Wd, n, m, g, vals, idx)])
    torch.cuda.synchronize()
    ok("k1 grouped sparsify", torch.equal(idx, i))
    # one launch over mixed classes: the lean body set, then the full one (n = 3, element-aligned rows)
    for specs in ([(64, 768, 2, 4, 4), (40, 800, 1, 10, 4), (32, 256, 2, 8, 8)],
                  [(64, 768, 2, 4, 4), (48, 96, 3, 6, 16), (30, 66, 1, 6, 5)]):
        probs, refs = [], []
        for k, (Mq, Kq, nq, mq, gq) in enumerate(specs):
            Wq = synthetic.weights(Mq, Kq, seed=50 + k)
            probs.append((dev(Wq, "f32", ld_multiple=1 if Kq % 4 else 4), nq, mq, gq,
                          torch.empty((Mq, Kq // mq * nq), device="cuda"),
                          torch.empty((Mq // gq, Kq // mq, nq), dtype=torch.uint8, device="cuda")))
            refs.append(oracle.sparsify(Wq, nq, mq, gq))
        sten.sparsify_grouped_nm_batched(probs)
        torch.cuda.synchronize()
        ok("k1 grouped sparsify mixed %d" % len(specs[1]),
           all(np.array_equal(p[5].cpu().numpy().reshape(r[1].shape), r[1]) and np.array_equal(p[4].cpu().numpy(), r[0])
               for p, r in zip(probs, refs)))
    D = sten.densify(v, i, n, m, g, K)
    torch.cuda.synchronize()
    ok("k2 densify", np.array_equal(D.cpu().numpy(), oracle.densify(v_ref, i_ref, n, m, g, K)))
v, i = sten.sparsify_grouped_nm(Wd, n, m, g)
if on("k3"):
    for tile in range(1, 8):
        for split in (1, 3):
            C = sten.spmm_grouped_nm(v, i, Bdv, n, m, g, plan=sten.make_plan(sten.ALGO_SIMT, split, tile))
            torch.cuda.synchronize()
            ok("k3 simt tile %d split %d" % (tile, split), rel_err(C, C_ref, Bd) <= 1e-5)
    probs = [(v, i, Bdv, n, m, g, torch.empty((M, N), device="cuda"))]
    nb = sten.batched_workspace_size(probs, [3], 2)
    ws = torch.zeros(nb // 4 + 4, device="cuda")
    sten.spmm_grouped_nm_batched_ex(probs, ws, [3], 2)
    torch.cuda.synchronize()
    ok("k3 grouped split-K workspace", rel_err(probs[0][6], C_ref, Bd) <= 1e-5)
    R = torch.zeros((M, N), device="cuda")
    C = sten.spmm_grouped_nm_epilogue(v, i, Bdv, n, m, g, bias=torch.zeros(M, device="cuda"), act=1, residual=R)
    torch.cuda.synchronize()
    ok("k3 epilogue", bool(torch.isfinite(C).all()))
Wb, Bb = synthetic.weights(128, 512, seed=3, dtype="bf16"), synthetic.activations(512, 256, seed=4, dtype="bf16")
vb_ref, ib_ref = oracle.sparsify(Wb, 2, 4, 64)
Cb_ref, Bbd = oracle.spmm(vb_ref, ib_ref, Bb, 2, 4, 64)
vb, ib = sten.sparsify_grouped_nm(dev(Wb, "bf16"), 2, 4, 64)
if on("k4"):
    C = sten.spmm_grouped_nm(vb, ib, dev(Bb, "bf16"), 2, 4, 64, out_dtype=torch.float32,
                             plan=sten.make_plan(sten.ALGO_MMA_SYNC, 1, 1))
    torch.cuda.synchronize()
    ok("k4 mma.sync", rel_err(C, Cb_ref, Bbd) <= 2e-2)
if on("k5"):
    C = sten.spmm_grouped_nm(vb, ib, dev(Bb, "bf16"), 2, 4, 64, out_dtype=torch.float32,
                             plan=sten.make_plan(sten.ALGO_TCGEN05, 1, 3))
    torch.cuda.synchronize()
    ok("k5 tcgen05", rel_err(C, Cb_ref, Bbd) <= 2e-2)
if on("k6"):
    v24, meta = sten.sp24_pack(vb, ib, 2, 4, 64, 512)
    for tile in (1, 2, 3, 4, 5):
        C = sten.spmm_sp24(v24, meta, 128, 512, dev(Bb, "bf16"), out_dtype=torch.float32, tile=tile)
        torch.cuda.synchronize()
        ok("k6 sp24 tile %d" % tile, rel_err(C, Cb_ref, Bbd) <= 2e-2)
if on("nmg"):
    Wn = synthetic.weights(16, 48, seed=5)
    Bn = synthetic.activations(48, 40, seed=6)
    for method in (0, 1, 2):
        vn, inn = sten.nmg_sparsify(dev(Wn, "f32"), 2, 4, 2, method=method)
        ref = oracle.nmg_sparsify(Wn, 2, 4, 2) if method == 0 else oracle.nmg_sparsify_exchange(Wn, 2, 4, 2, method - 1)
        torch.cuda.synchronize()
        ok("nmg convert %d" % method, np.array_equal(inn.cpu().numpy().view(np.uint16), ref[1]))
    vn, inn = sten.nmg_sparsify(dev(Wn, "f32"), 2, 4, 2)
    Cn = sten.nmg_spmm(vn, inn, dev(Bn, "f32"), 2, 4, 2)
    Cn_ref, Bn_b = oracle.nmg_spmm(*oracle.nmg_sparsify(Wn, 2, 4, 2), Bn, 2, 4, 2)
    torch.cuda.synchronize()
    ok("nmg spmm", rel_err(Cn, Cn_ref, Bn_b) <= 1e-5)
if on("masked"):
    G = synthetic.activations(M, N, seed=7)
    dV = sten.sddmm_grouped_nm(dev(G, "f32"), Bdv, i, n, m, g)
    dV_ref, bnd = oracle.sddmm(G, B, i_ref, n, m, g)
    torch.cuda.synchronize()
    ok("sddmm", rel_err(dV, dV_ref, bnd) <= 1e-5)
    vals, out = sten.mask_check_repack(sten.densify(v, i, n, m, g, K), i, n, m, g)
    torch.cuda.synchronize()
    ok("mask check", int(out.item()) == 0 and torch.equal(vals, v))
print("DONE", flush=True)
