"""GPU parity of the protocol layer through the C ABI:
keygen / sign / verify / ecdh on the B200 against golden vectors produced by the
compiled reference, the C oracle on fresh inputs, and size-independent round-trip
properties at 2^20 lanes."""
import hashlib
import random

import numpy as np
import pytest

import paper_2501_03245_b200 as gecc
from oracle import coracle as O
from oracle import pyec as E
from tests.util import CURVE_IDS, golden

pytestmark = pytest.mark.gpu
ECDSA = golden("ecdsa")
CURVES = ["sm2", "secp256k1"]


@pytest.fixture(scope="module")
def ctxs():
    c = {0: gecc.Context(gecc.SM2), 1: gecc.Context(gecc.SECP256K1)}
    yield c
    for x in c.values():
        x.close()


@pytest.mark.parametrize("name", CURVES)
def test_ecdsa_golden_gpu(ctxs, name):
    ent, cid, c = ECDSA[name], CURVE_IDS[name], E.CURVES[name]
    ctx = ctxs[cid]
    n = ent["n"]
    sec, pub = bytes.fromhex(ent["secrets"]), bytes.fromhex(ent["publics"])
    dig, sig = bytes.fromhex(ent["digests"]), bytes.fromhex(ent["sigs"])
    assert ctx.keygen(ent["keygen_seed"], n) == (0, sec, pub)
    assert ctx.sign(dig, sec, ent["nonce_seed"]) == (0, sig, [0] * n)
    # shard invariance: nonce stream = global lane index (protocol.cpp:125-126)
    assert ctx.sign(dig[32 * 8:], sec[32 * 8:], ent["nonce_seed"], lane_base=8)[1] == sig[64 * 8:]
    assert ctx.keygen(ent["keygen_seed"], n - 5, lane_base=5)[2] == pub[65 * 5:]
    for case in ent["verify_cases"]:  # perturbation matrix, malformed keys, Q = +-G, R = infinity
        d, p, sg = (bytes.fromhex(case[k]) for k in ("digests", "publics", "sigs"))
        rc, res = ctx.verify(d, p, sg)
        assert (rc, list(res)) == (0, case["results"]), case["name"]
    rt = ent["retry"]  # s == 0 on attempt 0 -> fresh nonce (test_protocol.cpp:196-228)
    rc, s, st = ctx.sign(bytes.fromhex(rt["digests"]), bytes.fromhex(rt["secrets"]), rt["nonce_seed"])
    assert (rc, s.hex(), st) == (0, rt["sigs"], [0, 0])
    # zero / oversize secret fails the whole call (test_capi.cpp:203-213)
    assert ctx.sign(dig[:64], bytes(32) + sec[32:64], 7)[0] == 2
    assert ctx.sign(dig[:64], E.be32(c.n) + sec[32:64], 7)[0] == 2
    eh = ent["ecdh"]
    rc, sh, st = ctx.ecdh(bytes.fromhex(eh["secrets"]), bytes.fromhex(eh["peers"]))
    assert (rc, sh.hex(), st) == (eh["rc"], eh["shared"], eh["status"])
    # lane_status == NULL -> first failing lane's code (capi.cpp:64-73)
    assert ctx.ecdh(bytes.fromhex(eh["secrets"]), bytes.fromhex(eh["peers"]), want_status=False)[0] == 3
    kb = ent["keybatch"]
    d = bytearray((kb["seed"] + 37 * i) & 0xFF for i in range(32 * kb["n"]))
    for i in range(kb["n"]):
        d[32 * i] = 0x13
    rc, ksec, kpub = ctx.keygen(kb["seed"], kb["n"])
    assert kpub.hex() == kb["publics"]
    assert ctx.sign(bytes(d), ksec, kb["nonce_seed"])[1].hex() == kb["sigs"]


@pytest.mark.parametrize("name", CURVES)
def test_ecdsa_bulk_digest_gpu(ctxs, name):
    """n = 1024 keygen+sign outputs hashed; digests recorded from the reference."""
    ent, ctx = ECDSA[name]["bulk1024"], ctxs[CURVE_IDS[name]]
    n = 1024
    rc, sec, pub = ctx.keygen(5, n)
    dig = b"".join(hashlib.sha256(i.to_bytes(8, "big")).digest() for i in range(n))
    rc, sig, st = ctx.sign(dig, sec, 7)
    assert rc == 0 and not any(st)
    assert hashlib.sha256(pub).hexdigest() == ent["publics_sha256"]
    assert hashlib.sha256(sig).hexdigest() == ent["sigs_sha256"]
    assert ctx.verify(dig, pub, sig) == (0, b"\x01" * n)


@pytest.mark.parametrize("cid", [0, 1])
def test_ecdsa_random_vs_oracle(ctxs, cid):
    ctx = ctxs[cid]
    rng = random.Random(700 + cid)
    n = 200
    rc, sec, pub = ctx.keygen(31 + cid, n)
    assert O.keygen(cid, 31 + cid, n) == (0, sec, pub)
    dig = bytes(rng.randrange(256) for _ in range(32 * n))
    got = ctx.sign(dig, sec, 99)
    assert got == O.ecdsa_sign(cid, dig, sec, 99)
    bad = bytearray(got[1])
    for i in range(0, n, 7):
        bad[64 * i + rng.randrange(64)] ^= 1 << rng.randrange(8)
    bp = bytearray(pub)
    for i in range(3, n, 11):
        bp[65 * i + 1 + rng.randrange(64)] ^= 1 << rng.randrange(8)
    assert ctx.verify(dig, bytes(bp), bytes(bad)) == O.ecdsa_verify(cid, dig, bytes(bp), bytes(bad))
    assert ctx.ecdh(sec, bytes(bp)) == O.ecdh(cid, sec, bytes(bp))


def test_ecdsa_api_edges(ctxs):
    ctx = ctxs[1]
    assert ctx.sign(b"", b"", 3)[:2] == (0, b"")          # empty batches (test_protocol.cpp:280-286)
    assert ctx.verify(b"", b"", b"") == (0, b"")
    assert ctx.keygen(3, 0) == (0, b"", b"")
    l = gecc.lib()
    assert l.sm2b_verify(ctx.h, 1, None, None, None, None) == 1   # NULL buffers with count > 0
    assert l.sm2b_sign(None, 0, None, None, 1, None, None) == 1   # NULL ctx
    # seed 0 = system entropy: two calls differ (test_capi.cpp:62-66)
    a = ctx.keygen(0, 1)[1]
    b = ctx.keygen(0, 1)[1]
    assert a != b
    # reference-compatible constructor: SM2, ledger economics pinned by test_capi.cpp:156-175
    with gecc.Context(reference_compat=True, workers=1) as sm2:
        assert sm2.curve == gecc.SM2
        rc, sec, pub = sm2.keygen(11, 8)
        sm2.ledger_reset()
        dig = bytes(range(32)) * 8
        sm2.sign(dig, sec, 23)
        assert sm2.ledger()["modinv"] == 257


def test_ecdsa_roundtrip_large(ctxs):
    """2^20 lanes on secp256k1: keygen -> sign -> verify all ones; one flipped bit per
    16th lane flips exactly those lanes; sharded signing == single call (checksum)."""
    ctx = ctxs[1]
    n = 1 << 20
    rc, sec, pub = ctx.keygen(2024, n)
    assert rc == 0
    rs = np.random.RandomState(5)
    dig = rs.bytes(32 * n)
    rc, sig, st = ctx.sign(dig, sec, 77)
    assert rc == 0 and not any(st)
    rc, res = ctx.verify(dig, pub, sig)
    assert rc == 0 and res == b"\x01" * n
    bad = np.frombuffer(sig, np.uint8).copy().reshape(n, 64)
    bad[::16, 37] ^= 0x20
    rc, res = ctx.verify(dig, pub, bad.tobytes())
    want = np.ones(n, np.uint8)
    want[::16] = 0
    assert rc == 0 and (np.frombuffer(res, np.uint8) == want).all()
    half = n // 2
    s0 = ctx.sign(dig[:32 * half], sec[:32 * half], 77, lane_base=0)[1]
    s1 = ctx.sign(dig[32 * half:], sec[32 * half:], 77, lane_base=half)[1]
    assert hashlib.sha256(s0 + s1).digest() == hashlib.sha256(sig).digest()
    # CPU spot check of 48 random lanes against the oracle
    for i in rs.choice(n, 48, replace=False):
        i = int(i)
        assert O.ecdsa_sign(1, dig[32 * i:32 * i + 32], sec[32 * i:32 * i + 32], 77, lane_base=i)[1] == sig[64 * i:64 * i + 64]


def test_bench_run_gpu(ctxs):
    """sm2b_bench_run: both strategies compared before timing (bench.cpp:253-256), ledger in the
    reference's closed forms (acceptance.cpp criteria 3 and 7), argument errors (capi.cpp:266-273)."""
    with gecc.Context(reference_compat=True, workers=1) as sm2:
        n = 512
        for op in ("padd", "fpmul", "upmul", "sign", "verify"):
            for strategy in ("affine-batch", "jacobian-serial"):
                rc, rep = sm2.bench_run(op, strategy, n, lanes=8, seed=1, repeats=3)
                assert rc == 0 and rep["equivalence_checked"] == 1, (op, strategy)
                assert rep["wall_seconds"] > 0 and rep["throughput"] > 0 and rep["lanes_used"] == 8
        rc, rep = sm2.bench_run("padd", "affine-batch", 4096, lanes=16, repeats=3)
        assert (rep["ops"]["modmul"], rep["ops"]["modsub"], rep["ops"]["modinv"]) == (6 * 4096 - 3, 6 * 4096, 1)
        assert rep["modeled_cost"] == 6 * 4096 + 5 * (6 * 4096 - 3) + 500
        rc, rep = sm2.bench_run("upmul", "affine-batch", 32, lanes=8, repeats=1)
        assert rep["ops"] == dict(modmul=120064, modadd=40960, modsub=90112, modinv=256)  # acceptance.cpp crit. 7
        assert sm2.bench_run("nope", "affine-batch", 8)[0] == 1
        assert sm2.bench_run("padd", "quantum", 8)[0] == 1
        assert sm2.bench_run("padd", "affine-batch", 0)[0] == 1
        assert sm2.bench_run("padd", "affine-batch", 8, repeats=0)[0] == 1
    rc, rep = ctxs[1].bench_run("verify", "affine-batch", 1 << 14, repeats=3)
    assert rc == 0 and rep["equivalence_checked"] == 1


@pytest.mark.parametrize("cid", [0, 1])
def test_sign_group_retry_and_ragged_gpu(ctxs, cid):
    """k_sign signs 4 lanes per thread with shared inversions: forced retry inside a group,
    ragged batch sizes (tail lanes), and a malformed secret inside a group."""
    c, ctx = E.CURVES[cid], ctxs[cid]
    rng = random.Random(199 + cid)
    n, seed, rig = 11, 13, 5
    sec = b"".join(E.be32(rng.randrange(1, c.n)) for _ in range(n))
    dig = bytearray(rng.randrange(256) for _ in range(32 * n))
    d = int.from_bytes(sec[32 * rig:32 * rig + 32], "big")
    r0 = E.ec_mul(c, E.nonce(c, seed, rig, 0), c.G)[0] % c.n
    dig[32 * rig:32 * rig + 32] = E.be32((-r0 * d) % c.n)
    want = O.ecdsa_sign(cid, bytes(dig), sec, seed)
    assert ctx.sign(bytes(dig), sec, seed) == want
    for m in (1, 2, 3, 4, 5, 7, 9):
        assert ctx.sign(bytes(dig[:32 * m]), sec[:32 * m], seed) == O.ecdsa_sign(cid, bytes(dig[:32 * m]), sec[:32 * m], seed)
    bad = bytearray(sec)
    bad[32 * 6:32 * 7] = bytes(32)
    assert ctx.sign(bytes(dig), bytes(bad), seed)[0] == 2
