"""Device-resident entry points (gecc_*_dev): torch tensors in, torch tensors out, work
enqueued on the caller's stream without synchronisation; results must equal the host-pointer
entry points' (which are parity-tested against the oracle)."""
import ctypes as C
import random

import numpy as np
import pytest
import torch

import paper_2501_03245_b200 as gecc
from oracle import coracle as O
from oracle import pyec as E

pytestmark = pytest.mark.gpu


def vp(t):
    return C.c_void_p(t.data_ptr())


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32 if a.dtype == np.uint32 else a.dtype)).cuda()


def host_u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("cid", [0, 1])
def test_dev_entry_points_match_host_api(cid):
    c = E.CURVES[cid]
    rng = random.Random(800 + cid)
    n = 777
    l = gecc.lib()
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream), gecc.Context(cid, 0) as ctx:
        ctx.set_stream(stream.cuda_stream)
        k1 = gecc.cols_from_ints([rng.randrange(1 << 256) for _ in range(n)])
        k2 = gecc.cols_from_ints([rng.randrange(1, c.n) for _ in range(n)])
        col = lambda: torch.empty((8, n), dtype=torch.int32, device="cuda")
        flag = lambda: torch.empty(n, dtype=torch.uint8, device="cuda")
        P, T, S = (col(), col(), flag()), (col(), col(), flag()), (col(), col(), flag())
        assert l.gecc_batch_fpmul_dev(ctx.h, C.c_size_t(n), vp(dev(k1)), vp(P[0]), vp(P[1]), vp(P[2])) == 0
        assert l.gecc_batch_fpmul_dev(ctx.h, C.c_size_t(n), vp(dev(k2)), vp(T[0]), vp(T[1]), vp(T[2])) == 0
        assert l.gecc_batch_padd_dev(ctx.h, C.c_size_t(n), vp(P[0]), vp(P[1]), vp(P[2]), vp(T[0]), vp(T[1]),
                                     vp(T[2]), vp(S[0]), vp(S[1]), vp(S[2])) == 0
        stream.synchronize()
        Ph = (host_u32(P[0]), host_u32(P[1]), P[2].cpu().numpy())
        Th = (host_u32(T[0]), host_u32(T[1]), T[2].cpu().numpy())
        Sh = (host_u32(S[0]), host_u32(S[1]), S[2].cpu().numpy())
        for a, b in zip(Ph, O.batch_fpmul(cid, k1)):
            assert (a == b).all()
        for a, b in zip(Sh, O.batch_padd(cid, Ph, Th)):
            assert (a == b).all()
        # pdbl / upmul / invert / msm
        D = (col(), col(), flag())
        assert l.gecc_batch_pdbl_dev(ctx.h, C.c_size_t(n), vp(P[0]), vp(P[1]), vp(P[2]), vp(D[0]), vp(D[1]), vp(D[2])) == 0
        m = 64
        sub = lambda A: tuple(a[..., :m].contiguous() for a in A)
        Pm, U = sub(P), (torch.empty((8, m), dtype=torch.int32, device="cuda"),
                         torch.empty((8, m), dtype=torch.int32, device="cuda"),
                         torch.empty(m, dtype=torch.uint8, device="cuda"))
        ks = np.ascontiguousarray(k2[:, :m])
        assert l.gecc_batch_upmul_dev(ctx.h, C.c_size_t(m), vp(dev(ks)), vp(Pm[0]), vp(Pm[1]), vp(Pm[2]), vp(U[0]),
                                      vp(U[1]), vp(U[2])) == 0
        inv_in = gecc.cols_from_ints([0 if i % 9 == 0 else rng.randrange(1, c.p) for i in range(n)])
        inv_out = col()
        assert l.gecc_batch_invert_dev(ctx.h, 0, C.c_size_t(n), vp(dev(inv_in)), vp(inv_out)) == 0
        M = (torch.empty((8, 1), dtype=torch.int32, device="cuda"), torch.empty((8, 1), dtype=torch.int32, device="cuda"),
             torch.empty(1, dtype=torch.uint8, device="cuda"))
        assert l.gecc_msm_dev(ctx.h, C.c_size_t(m), vp(dev(ks)), vp(Pm[0]), vp(Pm[1]), vp(Pm[2]), vp(M[0]), vp(M[1]), vp(M[2])) == 0
        stream.synchronize()
        for a, b in zip((host_u32(D[0]), host_u32(D[1]), D[2].cpu().numpy()), O.batch_pdbl(cid, Ph)):
            assert (a == b).all()
        Pmh = tuple(np.ascontiguousarray(a[..., :m]) for a in Ph)
        for a, b in zip((host_u32(U[0]), host_u32(U[1]), U[2].cpu().numpy()), O.pmul_serial(cid, ks, Pmh)):
            assert (a == b).all()
        assert (host_u32(inv_out) == O.batch_invert(cid, 0, inv_in)).all()
        for a, b in zip((host_u32(M[0]), host_u32(M[1]), M[2].cpu().numpy()), O.msm(cid, ks, Pmh)):
            assert (a == b).all()
        # byte-record kernels on device buffers
        rc, sec, pub = ctx.keygen(3, n)
        dig = bytes(rng.randrange(256) for _ in range(32 * n))
        u8 = lambda b: torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
        d_sig = torch.empty(64 * n, dtype=torch.uint8, device="cuda")
        d_st = torch.empty(n, dtype=torch.int32, device="cuda")
        d_res = torch.empty(n, dtype=torch.uint8, device="cuda")
        d_dig, d_sec, d_pub = u8(dig), u8(sec), u8(pub)
        assert l.gecc_sign_dev(ctx.h, C.c_size_t(n), vp(d_dig), vp(d_sec), C.c_uint64(5), C.c_uint64(40), vp(d_sig), vp(d_st)) == 0
        assert l.gecc_verify_dev(ctx.h, C.c_size_t(n), vp(d_dig), vp(d_pub), vp(d_sig), vp(d_res)) == 0
        stream.synchronize()
        assert bytes(d_sig.cpu().numpy()) == ctx.sign(dig, sec, 5, lane_base=40)[1]
        assert int(d_res.sum()) == n and int(d_st.abs().sum()) == 0
        # device signing refuses seed 0 (system entropy is a host-side service)
        assert l.gecc_sign_dev(ctx.h, C.c_size_t(n), vp(d_dig), vp(d_sec), C.c_uint64(0), C.c_uint64(0), vp(d_sig), vp(d_st)) == 7


def test_pipelined_host_api_matches_dev_api_on_a_large_ragged_batch():
    """The host entry points cut large batches into chunks (short head chunk, two compute streams,
    strided 2-D copies for column buffers); every byte must equal the single-launch device path.
    Size chosen to exercise the head chunk, unequal last chunk and a ragged tail."""
    n = (1 << 19) + (1 << 16) + 3
    l = gecc.lib()
    with gecc.Context(gecc.SECP256K1, 0) as ctx:
        rc, sec, pub = ctx.keygen(9, n)
        assert rc == 0
        dig = np.random.RandomState(5).bytes(32 * n)
        u8 = lambda b: torch.from_numpy(np.frombuffer(b, np.uint8).copy()).cuda()
        d_dig, d_sec, d_pub = u8(dig), u8(sec), u8(pub)
        d_sig = torch.empty(64 * n, dtype=torch.uint8, device="cuda")
        d_st = torch.empty(n, dtype=torch.int32, device="cuda")
        assert l.gecc_sign_dev(ctx.h, C.c_size_t(n), vp(d_dig), vp(d_sec), C.c_uint64(3), C.c_uint64(0), vp(d_sig), vp(d_st)) == 0
        torch.cuda.synchronize()
        rc, sig, st = ctx.sign(dig, sec, 3)
        assert rc == 0 and sig == d_sig.cpu().numpy().tobytes() and not any(st)
        # verify: flip a few lanes so that both outcomes travel through every chunk
        bad = bytearray(sig)
        flipped = [0, 1, 65535, 65536, 65537, n // 2, n - 1]
        for i in flipped:
            bad[64 * i + 40] ^= 1
        d_res = torch.empty(n, dtype=torch.uint8, device="cuda")
        assert l.gecc_verify_dev(ctx.h, C.c_size_t(n), vp(d_dig), vp(d_pub), vp(u8(bytes(bad))), vp(d_res)) == 0
        torch.cuda.synchronize()
        rc, res = ctx.verify(dig, pub, bytes(bad))
        assert rc == 0 and res == d_res.cpu().numpy().tobytes()
        assert sum(res) == n - len(flipped) and all(res[i] == 0 for i in flipped)
        # a malformed secret in the LAST chunk fails the whole call before any output is written
        broken = bytearray(sec)
        broken[32 * (n - 2):32 * (n - 1)] = bytes(32)
        rc, sig2, _ = ctx.sign(dig, bytes(broken), 3)
        assert rc == 2 and sig2 == bytes(64 * n)
        # column buffers: padd through the chunked host path vs the device path
        k = np.random.RandomState(6).randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32)
        P = ctx.batch_fpmul(k)
        T = ctx.batch_fpmul(np.ascontiguousarray(k[::-1]))
        S = ctx.batch_padd(P, T)
        dP, dT = tuple(dev(a) for a in P), tuple(dev(a) for a in T)
        dS = (torch.empty((8, n), dtype=torch.int32, device="cuda"), torch.empty((8, n), dtype=torch.int32, device="cuda"),
              torch.empty(n, dtype=torch.uint8, device="cuda"))
        assert l.gecc_batch_padd_dev(ctx.h, C.c_size_t(n), vp(dP[0]), vp(dP[1]), vp(dP[2]), vp(dT[0]), vp(dT[1]), vp(dT[2]),
                                     vp(dS[0]), vp(dS[1]), vp(dS[2])) == 0
        torch.cuda.synchronize()
        assert (S[0] == host_u32(dS[0])).all() and (S[1] == host_u32(dS[1])).all() and (S[2] == dS[2].cpu().numpy()).all()
        led0 = ctx.ledger()
        ctx.batch_padd(P, T)
        led1 = ctx.ledger()
        assert led1["modinv"] - led0["modinv"] == 1 and led1["modmul"] - led0["modmul"] == 6 * n - 3  # one call, one closed form
