#!/usr/bin/env python
"""BASELINE.json configs[4]: batch-size sweep 2^12 .. 2^24 for ECDSA verify and batched
point addition on one GPU, next to the CPU reference (oracle/_ref, all host threads) at
n <= 2^16 (its throughput is flat beyond ~2^12).  Writes gpurun_out/sweep.json.

Device-resident timing with CUDA events (median of 5 after one warm-up, as bench.cpp:262-281),
inputs generated on the GPU with the library's own keygen / sign / fixed-base kernels.
"""
import ctypes as C
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_03245_b200 as gecc  # noqa: E402


def timed(fn, stream, repeats=5):
    fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    return statistics.median(ms)


def main():
    lo, hi = 12, int(os.environ.get("SWEEP_MAX_LOG2", "24"))
    ctx = gecc.Context(gecc.SECP256K1, 0)
    l = gecc.lib()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    vp = lambda t: C.c_void_p(t.data_ptr())
    u8 = lambda m: torch.empty(m, dtype=torch.uint8, device="cuda")
    nmax = 1 << hi
    # records for the largest size once; smaller sizes use prefixes
    d_sec, d_pub, d_sig, d_res = u8(32 * nmax), u8(65 * nmax), u8(64 * nmax), u8(nmax)
    d_st = torch.empty(nmax, dtype=torch.int32, device="cuda")
    d_dig = torch.randint(0, 256, (32 * nmax,), dtype=torch.uint8, device="cuda")
    h_sec, h_pub = np.empty(32 * nmax, np.uint8), np.empty(65 * nmax, np.uint8)
    assert l.gecc_keygen(ctx.h, C.c_uint64(1), C.c_uint64(0), C.c_size_t(nmax), C.c_void_p(h_sec.ctypes.data),
                         C.c_void_p(h_pub.ctypes.data)) == 0
    d_sec.copy_(torch.from_numpy(h_sec))
    d_pub.copy_(torch.from_numpy(h_pub))
    assert l.gecc_sign_dev(ctx.h, C.c_size_t(nmax), vp(d_dig), vp(d_sec), C.c_uint64(7), C.c_uint64(0), vp(d_sig),
                           vp(d_st)) == 0
    torch.cuda.synchronize()
    col = lambda: torch.empty((8, nmax), dtype=torch.int32, device="cuda")
    k = torch.randint(-2**31, 2**31 - 1, (8, nmax), dtype=torch.int32, device="cuda")
    P = (col(), col(), u8(nmax)); T = (col(), col(), u8(nmax)); S = (col(), col(), u8(nmax))
    l.gecc_batch_fpmul_dev(ctx.h, C.c_size_t(nmax), vp(k), vp(P[0]), vp(P[1]), vp(P[2]))
    k2 = torch.randint(-2**31, 2**31 - 1, (8, nmax), dtype=torch.int32, device="cuda")
    l.gecc_batch_fpmul_dev(ctx.h, C.c_size_t(nmax), vp(k2), vp(T[0]), vp(T[1]), vp(T[2]))
    torch.cuda.synchronize()
    rows = []
    from oracle import refshim as gate_mod   # checker only: the compiled reference, per-size parity gates
    gate = gate_mod if gate_mod.available() else None
    for lg in range(lo, hi + 1, 2):
        n = 1 << lg
        # column buffers must be contiguous per size: repack the prefix (limb k at k*n + i)
        sub = lambda A: tuple(a[:, :n].contiguous() if a.dim() == 2 else a[:n].contiguous() for a in A)
        Pn, Tn, Sn = sub(P), sub(T), sub(S)
        ms_v = timed(lambda: l.gecc_verify_dev(ctx.h, C.c_size_t(n), vp(d_dig), vp(d_pub), vp(d_sig), vp(d_res)), stream)
        assert int(d_res[:n].sum()) == n
        # parity gate of this size (verify): a sample of lanes, two of them forged, through the CPU
        # reference (oracle/_ref) and the GPU -- the same verdict lane by lane
        if gate is not None:
            m = min(n, 256)
            idx = np.linspace(0, n - 1, m).astype(np.int64)
            take = lambda d, w: d.view(-1, w)[torch.from_numpy(idx).cuda()].contiguous()
            g_dig, g_pub, g_sig = take(d_dig[:32 * n], 32), take(d_pub[:65 * n], 65), take(d_sig[:64 * n], 64).clone()
            g_sig[3, 5] ^= 1
            g_sig[m - 1, 40] ^= 0x80
            g_res = u8(m)
            assert l.gecc_verify_dev(ctx.h, C.c_size_t(m), vp(g_dig), vp(g_pub), vp(g_sig), vp(g_res)) == 0
            rc, want = gate.ecdsa_verify(1, g_dig.cpu().numpy().tobytes(), g_pub.cpu().numpy().tobytes(),
                                         g_sig.cpu().numpy().tobytes(), workers=0)
            assert rc == 0 and g_res.cpu().numpy().tobytes() == want and want.count(b"\x00") == 2, f"verify parity at 2^{lg}"
        padd = lambda: l.gecc_batch_padd_dev(ctx.h, C.c_size_t(n), vp(Pn[0]), vp(Pn[1]), vp(Pn[2]), vp(Tn[0]),
                                             vp(Tn[1]), vp(Tn[2]), vp(Sn[0]), vp(Sn[1]), vp(Sn[2]))
        forms = {}
        outs = {}
        for name in ("chunked", "coop128", "tiled8", "fused", "auto"):  # one inversion per thread / per block / per tile; library's pick
            gecc.set_batch_form(name)
            forms[name] = timed(padd, stream)
            outs[name] = tuple(t.clone() for t in Sn)
        gecc.set_batch_form("auto")
        ms_p = forms["auto"]
        # parity gate of this size (padd): every form gives the same bytes for ALL n pairs, and a sample
        # of the pairs (all of them up to 2^16) equals the CPU reference's batch_padd
        for name, o in outs.items():
            assert all(bool((a == b).all()) for a, b in zip(o, outs["chunked"])), f"padd form {name} differs at 2^{lg}"
        if gate is not None:
            m = min(n, 1 << 16)
            idx = torch.from_numpy(np.linspace(0, n - 1, m).astype(np.int64)).cuda()
            pick = lambda A: tuple((a[:, idx] if a.dim() == 2 else a[idx]).contiguous().cpu().numpy() for a in A)
            as_u = lambda A: (A[0].view(np.uint32), A[1].view(np.uint32), A[2])
            want = gate.batch_padd(1, as_u(pick(Pn)), as_u(pick(Tn)), workers=0)
            got = as_u(pick(outs["auto"]))
            assert all((np.asarray(w) == g).all() for w, g in zip(want, got)), f"padd parity at 2^{lg}"
        rows.append(dict(log2n=lg, verify_ms=ms_v, verify_per_s=n / ms_v * 1e3, padd_ms=ms_p, padd_per_s=n / ms_p * 1e3,
                         padd_ms_by_form=forms))
        print(f"2^{lg:2d}  verify {ms_v:9.3f} ms  {n / ms_v / 1e3:8.2f} M/s   padd {ms_p:8.4f} ms  {n / ms_p / 1e6:7.3f} G/s"
              "  (" + ", ".join(f"{k} {v:.4f}" for k, v in forms.items()) + ")", flush=True)
    # CPU reference at 2^12, 2^14, 2^16
    cpu = []
    from oracle import refshim as R
    if R.available() and not os.environ.get("SWEEP_NO_CPU"):
        h_dig, h_sig = d_dig[:32 << 16].cpu().numpy().tobytes(), d_sig[:64 << 16].cpu().numpy().tobytes()
        Pc = tuple(a.cpu().numpy().view(np.uint32 if a.dim() == 2 else np.uint8) for a in sub_cpu(P, 1 << 16))
        Tc = tuple(a.cpu().numpy().view(np.uint32 if a.dim() == 2 else np.uint8) for a in sub_cpu(T, 1 << 16))
        for lg in (12, 14, 16):
            n = 1 << lg
            t0 = time.perf_counter()
            rc, res = R.ecdsa_verify(1, h_dig[:32 * n], h_pub[:65 * n].tobytes(), h_sig[:64 * n], workers=0)
            dt = time.perf_counter() - t0
            assert res == b"\x01" * n
            cut = lambda A: tuple(np.ascontiguousarray(a[..., :n]) for a in A)
            tp = R.batch_padd_timed(1, cut(Pc), cut(Tc), workers=0, repeats=3)
            cpu.append(dict(log2n=lg, verify_per_s=n / dt, padd_per_s=n / tp, cores=os.cpu_count()))
            print(f"CPU 2^{lg}: verify {n / dt:9.0f}/s  padd {n / tp / 1e6:6.2f} M/s  ({os.cpu_count()} cores)", flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/sweep.json", "w") as f:
        json.dump(dict(gpu=rows, cpu_reference=cpu, curve="secp256k1",
                       parity="every size: verify sample (two forged lanes) and padd (all forms equal; sample of <= 2^16 pairs) checked against oracle/_ref"
                       if gate is not None else "oracle/_ref not built: sizes unchecked"), f, indent=1)


def sub_cpu(A, n):
    return tuple(a[:, :n].contiguous() if a.dim() == 2 else a[:n].contiguous() for a in A)


if __name__ == "__main__":
    main()
