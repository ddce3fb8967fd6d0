#!/usr/bin/env python
"""Experiment: device-resident batch_padd time per kernel form and size (median of 7), with the
outputs of every form compared with the chunked form's."""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2501_03245_b200 as gecc

forms = sys.argv[1].split(",") if len(sys.argv) > 1 else ["chunked", "coop128", "tiled8", "fused", "fused2"]
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [12, 14, 16, 18, 20, 22]
curve = gecc.SM2 if os.environ.get("CURVE") == "sm2" else gecc.SECP256K1
ctx = gecc.Context(curve, 0)
l = gecc.lib()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())
nmax = 1 << max(sizes)
rs = np.random.RandomState(5)
k = [torch.from_numpy(rs.randint(0, 2**32, size=(8, nmax), dtype=np.uint64).astype(np.uint32)).cuda() for _ in range(2)]
for log2n in sizes:
    n = 1 << log2n
    col = lambda: torch.empty((8, n), dtype=torch.int32, device="cuda")
    u8 = lambda: torch.zeros(n, dtype=torch.uint8, device="cuda")
    P, T = (col(), col(), u8()), (col(), col(), u8())
    for kk, X in zip(k, (P, T)):
        ks = kk[:, :n].contiguous()
        assert l.gecc_batch_fpmul_dev(ctx.h, C.c_size_t(n), vp(ks), vp(X[0]), vp(X[1]), vp(X[2])) == 0
    # a few exceptional lanes
    T[0][:, 5] = P[0][:, 5]; T[1][:, 5] = P[1][:, 5]
    P[2][9] = 1; P[0][:, 9] = 0; P[1][:, 9] = 0
    torch.cuda.synchronize()
    ref = None
    line = [f"2^{log2n:2d}"]
    for form in forms:
        gecc.set_batch_form(form)
        S = (col(), col(), u8())
        call = lambda: l.gecc_batch_padd_dev(ctx.h, C.c_size_t(n), vp(P[0]), vp(P[1]), vp(P[2]), vp(T[0]), vp(T[1]), vp(T[2]),
                                             vp(S[0]), vp(S[1]), vp(S[2]))
        for _ in range(3):
            assert call() == 0
        torch.cuda.synchronize()
        ms = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            assert call() == 0
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        got = tuple(t.clone() for t in S)
        if ref is None:
            ref = got
        ok = all(bool((a == b).all()) for a, b in zip(ref, got))
        t = statistics.median(ms)
        line.append(f"{form}: {t*1e3:8.1f} us {n/t/1e6:8.1f} G/s {'ok' if ok else 'MISMATCH'}")
    print(" | ".join(line), flush=True)
gecc.set_batch_form("auto")
