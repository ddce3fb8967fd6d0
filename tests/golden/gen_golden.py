#!/usr/bin/env python
"""Generates tests/golden/*.json from the compiled, unmodified reference
(oracle/_ref/libgecc_ref.so, built by `make -C oracle ref` from /root/reference).

Run in the authoring container only (needs /root/reference to build _ref):
    python tests/golden/gen_golden.py
The JSON files are committed; tests read them everywhere (also on the GPU box,
where /root/reference does not exist).

Inputs lifted from the reference's own tests (SURVEY.md section 8c "Fixtures"):
  * exceptional-lane set 3/7/11/19/23/31/47 in n=64      test_batch_point.cpp:70-100
  * zero masking incl. an all-zero batch                   test_batch_invert.cpp:147-170
  * reduce edge values                                     test_field.cpp:136-164
  * scalar edge set {0, 1, 2^77, n-1, all-ones raw}        test_batch_point.cpp:174-208
  * KeyBatch digest pattern                                test_capi.cpp:25-33
  * perturbation matrix for verify                         test_protocol.cpp:67-104
  * malformed C-ABI inputs                                 test_capi.cpp:97-111,203-213
"""
import hashlib
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import pyec as E  # noqa: E402
from oracle import refshim as R  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
H = lambda v: format(int(v), "064x")


def hx(cols):
    return [H(v) for v in R.cols_to_ints(cols)]


def pts_hex(P):
    return dict(x=hx(P[0]), y=hx(P[1]), inf=[int(v) for v in P[2]])


def gen_field():
    rng = random.Random(0xF1E1D)
    out = {}
    for cid in (0, 1):
        c = E.CURVES[cid]
        for which, q in ((0, c.p), (1, c.n)):
            fp = R.field_params(cid, which)
            edge = [0, 1, 2, q - 1, q - 2, (1 << 255) % q, fp["r"], fp["r2"], (q - 1) // 2]
            a = edge + [rng.randrange(q) for _ in range(40)]
            b = list(reversed(edge)) + [rng.randrange(q) for _ in range(40)]
            A, B = R.ints_to_cols(a), R.ints_to_cols(b)
            ent = dict(q=H(q), q_inv=fp["q_inv"], r=H(fp["r"]), r2=H(fp["r2"]), a=[H(v) for v in a],
                       b=[H(v) for v in b])
            for op in ("mont_mul", "mod_add", "mod_sub", "to_mont", "from_mont", "mod_inv"):
                ent[op] = hx(R.field_op(cid, which, op, A, B))
            # 512-bit reduce edges (test_field.cpp:136-141,153-164): c < q*2^256
            T = [q * (1 << 256) - 1, q * ((1 << 256) - 1), (q - 1) << 256, 1 << 256, 0, 1,
                 (1 << 256) - 1, ((q - 1) * (q - 1))]
            T += [rng.randrange(q << 256) for _ in range(24)]
            c16 = np.zeros((16, len(T)), np.uint32)
            for i, t in enumerate(T):
                for k in range(16):
                    c16[k, i] = (t >> (32 * k)) & 0xFFFFFFFF
            ent["reduce_in"] = [format(t, "0128x") for t in T]
            ent["reduce_generic"] = hx(R.mont_reduce(cid, which, c16, False))
            if cid == 0 and which == 0:
                ent["reduce_sm2"] = hx(R.mont_reduce(cid, which, c16, True))
            out[f"{c.name}.{'p' if which == 0 else 'n'}"] = ent
    return out


def mont_pts(cid, pts):
    """affine int points (or None) -> Montgomery-form column buffers"""
    c = E.CURVES[cid]
    fp = R.field_params(cid, 0)
    xs = [0 if p is None else p[0] * fp["r"] % c.p for p in pts]
    ys = [0 if p is None else p[1] * fp["r"] % c.p for p in pts]
    inf = np.array([1 if p is None else 0 for p in pts], np.uint8)
    return R.ints_to_cols(xs), R.ints_to_cols(ys), inf


def gen_batch():
    out = {}
    for cid in (0, 1):
        c = E.CURVES[cid]
        rng = random.Random(0xBA7C4 + cid)
        n = 64
        k1 = [rng.randrange(1, c.n) for _ in range(n)]
        k2 = [rng.randrange(1, c.n) for _ in range(n)]
        P = list(R.batch_fpmul(cid, R.ints_to_cols(k1), lanes=8))
        T = list(R.batch_fpmul(cid, R.ints_to_cols(k2), lanes=8))

        def setpt(dst, i, src, j, neg=False):
            dst[0][:, i] = src[0][:, j]
            dst[1][:, i] = src[1][:, j]
            dst[2][i] = src[2][j]
            if neg:
                y = R.cols_to_ints(src[1][:, j:j + 1])[0]
                dst[1][:, i] = R.ints_to_cols([(c.p - y) % c.p])[:, 0]

        def setinf(dst, i):
            dst[0][:, i] = 0
            dst[1][:, i] = 0
            dst[2][i] = 1

        setpt(T, 3, P, 3)            # doubling pair
        setpt(T, 7, P, 7, neg=True)  # inverse pair
        setinf(P, 11)
        setinf(T, 19)
        setinf(P, 23); setinf(T, 23)
        setpt(T, 31, P, 31)
        setinf(P, 47)
        ent = dict(k1=[H(v) for v in k1], k2=[H(v) for v in k2], P=pts_hex(P), T=pts_hex(T))
        ent["padd"] = pts_hex(R.batch_padd(cid, P, T, lanes=4))
        ent["pdbl"] = pts_hex(R.batch_pdbl(cid, P, lanes=4))
        # batch_invert with zeros (F_p and F_n) and an all-zero batch
        for which, q in ((0, c.p), (1, c.n)):
            vals = [rng.randrange(1, q) for _ in range(40)]
            for z in (0, 5, 17, 39):
                vals[z] = 0
            A = R.ints_to_cols(vals)
            ent[f"inv_in_{which}"] = [H(v) for v in vals]
            ent[f"inv_out_{which}"] = hx(R.batch_invert(cid, which, A, lanes=3))
        Z = np.zeros((8, 5), np.uint32)
        assert not R.batch_invert(cid, 0, Z, lanes=2).any()
        # scalar edge set, raw unreduced all-ones included (acceptance.cpp:288-291)
        edge = [0, 1, 2, 1 << 77, c.n - 1, c.n - 2, (1 << 256) - 1, c.n, c.n + 1, (1 << 255)]
        edge += [rng.randrange(1 << 256) for _ in range(6)]
        S = R.ints_to_cols(edge)
        ent["edge_scalars"] = [H(v) for v in edge]
        ent["fpmul_edge"] = pts_hex(R.batch_fpmul(cid, S, lanes=4))
        m = len(edge)
        Q = [np.ascontiguousarray(P[0][:, :m]), np.ascontiguousarray(P[1][:, :m]),
             np.ascontiguousarray(P[2][:m])]
        Q[2][5] = 1; Q[0][:, 5] = 0; Q[1][:, 5] = 0   # infinity input stays infinity
        ent["upmul_Q"] = pts_hex(Q)
        ent["upmul_edge"] = pts_hex(R.batch_upmul(cid, S, Q, lanes=4))
        ent["nonce"] = [[s, st, at, H(R.nonce(cid, s, st, at))]
                        for (s, st, at) in [(1, 0, 0), (1, 1, 0), (1, 0, 1), (7, 12345, 3),
                                            (0xDEADBEEF, 2**40 + 5, 7), (2**64 - 1, 2**63, 0)]]
        out[c.name] = ent
    return out


def keybatch_digests(n, seed):
    d = bytearray((seed + 37 * i) & 0xFF for i in range(32 * n))  # test_capi.cpp:25-33
    for i in range(n):
        d[32 * i] = 0x13
    return bytes(d)


def gen_ecdsa():
    out = {}
    ctx = R.Sm2bCtx(workers=4)
    for cid in (0, 1):
        c = E.CURVES[cid]
        ent = {}
        n = 24
        rc, sec, pub = R.keygen(cid, 5, n)
        assert rc == 0
        if cid == 0:
            assert (0, sec, pub) == ctx.keygen(5, n)
        dig = b"".join(hashlib.sha256(i.to_bytes(8, "big")).digest() for i in range(n))
        rc, sig, st = R.ecdsa_sign(cid, dig, sec, 7)
        assert rc == 0 and not any(st)
        if cid == 0:
            assert (0, sig, st) == ctx.sign(dig, sec, 7)
        ent.update(n=n, keygen_seed=5, nonce_seed=7, secrets=sec.hex(), publics=pub.hex(),
                   digests=dig.hex(), sigs=sig.hex())
        # perturbation matrix (test_protocol.cpp:67-104): each row is (digests, publics, sigs)
        cases = []

        def add_case(name, d, p, s):
            rc, res = R.ecdsa_verify(cid, d, p, s)
            assert rc == 0
            if cid == 0:
                assert (0, res) == ctx.verify(d, p, s), name
            cases.append(dict(name=name, digests=d.hex(), publics=p.hex(), sigs=s.hex(),
                              results=list(res)))

        add_case("valid", dig, pub, sig)
        bd = bytearray(dig); bd[32 * 2 + 31] ^= 1
        add_case("digest bit flipped lane 2", bytes(bd), pub, sig)
        bs = bytearray(sig); bs[64 * 3 + 5] ^= 0x10
        add_case("r perturbed lane 3", dig, pub, bytes(bs))
        bs = bytearray(sig); bs[64 * 4 + 40] ^= 0x10
        add_case("s perturbed lane 4", dig, pub, bytes(bs))
        bp = bytearray(pub); bp[65 * 5:65 * 6] = pub[65 * 6:65 * 7]
        add_case("wrong key lane 5", dig, bytes(bp), sig)
        bs = bytearray(sig); bs[64 * 6:64 * 6 + 32] = bytes(32)
        add_case("r = 0 lane 6", dig, pub, bytes(bs))
        bs = bytearray(sig); bs[64 * 7:64 * 7 + 32] = E.be32(c.n)
        add_case("r = n lane 7", dig, pub, bytes(bs))
        bs = bytearray(sig); bs[64 * 8 + 32:64 * 9] = E.be32(c.n)
        add_case("s = n lane 8", dig, pub, bytes(bs))
        bs = bytearray(sig); bs[64 * 8 + 32:64 * 9] = bytes(32)
        add_case("s = 0 lane 8", dig, pub, bytes(bs))
        bp = bytearray(pub); bp[65 * 9] = 0x05
        add_case("bad tag lane 9", dig, bytes(bp), sig)
        bp = bytearray(pub); bp[65 * 10 + 64] ^= 1
        add_case("off-curve key lane 10", dig, bytes(bp), sig)
        bp = bytearray(pub); bp[65 * 11 + 1:65 * 11 + 33] = E.be32(c.p)
        add_case("x = p lane 11", dig, bytes(bp), sig)
        # digest >= n is reduced, not rejected (capi.cpp:81-88): sign e, verify e+n
        e_small = 12345
        d_big = E.be32(e_small + c.n)
        rc, sg, _ = R.ecdsa_sign(cid, E.be32(e_small), sec[:32], 9)
        add_case("digest e+n equals e", d_big, pub[:65], sg)
        # Q = G and Q = -G (u1*G + u2*Q hits doubling / cancellation paths)
        for name, d in (("Q=G", 1), ("Q=-G", c.n - 1), ("d=2", 2)):
            q = E.encode_point(E.ec_mul(c, d, c.G))
            rc, sg, _ = R.ecdsa_sign(cid, dig[:32], E.be32(d), 11)
            add_case(name, dig[:32], q, sg)
        # forged: u1*G + u2*Q = infinity  (r arbitrary, choose e = -r*d so R = inf)
        d0 = int.from_bytes(sec[:32], "big")
        r0 = 0x1234567
        e0 = (-r0 * d0) % c.n
        add_case("R = infinity", E.be32(e0), pub[:65], E.be32(r0) + E.be32(1))
        ent["verify_cases"] = cases

        # s == 0 on attempt 0 forces a retry with a fresh nonce (test_protocol.cpp:196-228):
        # choose e = -r*d mod n for the attempt-0 nonce of stream 0.
        k0 = R.nonce(cid, 13, 0, 0)
        r0 = E.ec_mul(c, k0, c.G)[0] % c.n
        e0 = (-r0 * d0) % c.n
        rc, sg, st = R.ecdsa_sign(cid, E.be32(e0) + dig[32:64], sec[:64], 13)
        assert rc == 0 and st == [0, 0]
        k1 = R.nonce(cid, 13, 0, 1)
        assert sg[:32] == E.be32(E.ec_mul(c, k1, c.G)[0] % c.n)
        if cid == 0:
            assert (0, sg, st) == ctx.sign(E.be32(e0) + dig[32:64], sec[:64], 13)
        ent["retry"] = dict(nonce_seed=13, digests=(E.be32(e0) + dig[32:64]).hex(),
                            secrets=sec[:64].hex(), sigs=sg.hex())
        # lane_base: lanes 8.. signed as a shard starting at 8 equal the full batch
        rc, sg2, _ = R.ecdsa_sign(cid, dig[32 * 8:], sec[32 * 8:], 7, lane_base=8)
        assert sg2 == sig[64 * 8:]
        # malformed secrets fail the whole call (test_capi.cpp:203-213)
        ent["sign_zero_secret_rc"] = R.ecdsa_sign(cid, dig[:64], bytes(32) + sec[32:64], 7)[0]
        ent["sign_big_secret_rc"] = R.ecdsa_sign(cid, dig[:64], E.be32(c.n) + sec[32:64], 7)[0]
        # ECDH incl. invalid peer and zero secret (degenerate)
        peers = bytearray(pub[65:65 * 9] + pub[:65])
        peers[65 * 2 + 64] ^= 1
        secs = bytearray(sec[:32 * 9])
        secs[32 * 4:32 * 5] = bytes(32)
        rc, sh, st = R.ecdh(cid, bytes(secs), bytes(peers))
        if cid == 0:
            assert (rc, sh, st) == ctx.ecdh(bytes(secs), bytes(peers))
        ent["ecdh"] = dict(secrets=bytes(secs).hex(), peers=bytes(peers).hex(), shared=sh.hex(),
                           status=st, rc=rc)
        # bulk digests: n = 1024, sha256 over outputs
        nb = 1024
        rc, bsec, bpub = R.keygen(cid, 5, nb, workers=0)
        bdig = b"".join(hashlib.sha256(i.to_bytes(8, "big")).digest() for i in range(nb))
        rc, bsig, bst = R.ecdsa_sign(cid, bdig, bsec, 7, workers=0)
        rc, bres = R.ecdsa_verify(cid, bdig, bpub, bsig, workers=0)
        assert bres == b"\x01" * nb
        ent["bulk1024"] = dict(publics_sha256=hashlib.sha256(bpub).hexdigest(),
                               sigs_sha256=hashlib.sha256(bsig).hexdigest())
        # KeyBatch pattern
        kd = keybatch_digests(8, 17)
        rc, ksec, kpub = R.keygen(cid, 17, 8)
        rc, ksig, _ = R.ecdsa_sign(cid, kd, ksec, 23)
        ent["keybatch"] = dict(seed=17, nonce_seed=23, n=8, sigs=ksig.hex(), publics=kpub.hex())
        out[c.name] = ent
    # the survey's recorded values for SM2 must reproduce
    assert out["sm2"]["bulk1024"]["publics_sha256"] == \
        "5aff9204c91a70d134d02a4fd7bc524754a7496199148c15ab884280bff21b4c"
    assert out["sm2"]["bulk1024"]["sigs_sha256"] == \
        "60ad206ee25932b508adaafb0886c47260a1b5a9c0a54f1009d3bf905cbf0dbc"
    return out


def main():
    for name, fn in (("field", gen_field), ("batch", gen_batch), ("ecdsa", gen_ecdsa)):
        data = fn()
        data["_generated_by"] = "tests/golden/gen_golden.py from oracle/_ref (unmodified reference)"
        with open(os.path.join(OUT, f"{name}.json"), "w") as f:
            json.dump(data, f, indent=0, separators=(",", ":"))
        print(name, os.path.getsize(os.path.join(OUT, f"{name}.json")), "bytes")


if __name__ == "__main__":
    main()
