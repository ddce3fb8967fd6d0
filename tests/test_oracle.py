"""CPU tests of the checkers themselves (run everywhere, no GPU):

* the plain-C restatement (oracle/gecc_oracle.c) against every committed golden
  vector generated from the unmodified reference (tests/golden/gen_golden.py);
* the same restatement against the live compiled reference (oracle/_ref) on fresh
  random inputs, when _ref is present (marker `ref`);
* the independent Python-int oracle (oracle/pyec.py) against both.
"""
import hashlib
import random

import numpy as np
import pytest

from oracle import coracle as O
from oracle import pyec as E
from oracle import refshim as R
from tests.util import (CURVE_IDS, cols_hex, golden, hex_cols, pts_from_hex, pts_to_hex,
                        wide_cols)

FIELD = golden("field")
BATCH = golden("batch")
ECDSA = golden("ecdsa")
CURVES = ["sm2", "secp256k1"]


# ------------------------------------------------------------------ field
@pytest.mark.parametrize("key", [k for k in FIELD if not k.startswith("_")])
def test_field_golden(key):
    ent = FIELD[key]
    cid = CURVE_IDS[key.split(".")[0]]
    which = 0 if key.endswith(".p") else 1
    fp = O.field_params(cid, which)
    assert format(fp["q"], "064x") == ent["q"] and fp["q_inv"] == ent["q_inv"]
    assert format(fp["r"], "064x") == ent["r"] and format(fp["r2"], "064x") == ent["r2"]
    A, B = hex_cols(ent["a"]), hex_cols(ent["b"])
    for op in ("mont_mul", "mod_add", "mod_sub", "to_mont", "from_mont", "mod_inv"):
        assert cols_hex(O.field_op(cid, which, op, A, B)) == ent[op], op
    c16 = wide_cols(ent["reduce_in"])
    assert cols_hex(O.mont_reduce(cid, which, c16, False)) == ent["reduce_generic"]
    if "reduce_sm2" in ent:
        assert cols_hex(O.mont_reduce(cid, which, c16, True)) == ent["reduce_sm2"]
        assert ent["reduce_sm2"] == ent["reduce_generic"]  # test_field.cpp:166-169
        assert ent["q_inv"] == 1                            # test_field.cpp:27


def test_field_python_ints():
    """mont_mul(a,b) == a*b*R^-1 mod q, checked with Python ints (independent)."""
    for key, ent in FIELD.items():
        if key.startswith("_"):
            continue
        q = int(ent["q"], 16)
        rinv = pow(1 << 256, -1, q)
        for a, b, m, s, d in zip(ent["a"], ent["b"], ent["mont_mul"], ent["mod_add"], ent["mod_sub"]):
            a, b = int(a, 16), int(b, 16)
            assert int(m, 16) == a * b * rinv % q
            assert int(s, 16) == (a + b) % q and int(d, 16) == (a - b) % q
        for t, r in zip(ent["reduce_in"], ent["reduce_generic"]):
            assert int(r, 16) == int(t, 16) * rinv % q


# ------------------------------------------------------------------ batch
@pytest.mark.parametrize("name", CURVES)
def test_batch_golden(name):
    ent, cid = BATCH[name], CURVE_IDS[name]
    P, T = pts_from_hex(ent["P"]), pts_from_hex(ent["T"])
    for lanes in (1, 4, 7, 64):  # lane-count invariance (batch_invert.hpp:59-60)
        assert pts_to_hex(O.batch_padd(cid, P, T, lanes=lanes)) == ent["padd"]
        assert pts_to_hex(O.batch_pdbl(cid, P, lanes=lanes)) == ent["pdbl"]
    for i in (7, 23):
        assert ent["padd"]["inf"][i] == 1
    assert ent["padd"]["x"][3] == ent["pdbl"]["x"][3]
    for which in (0, 1):
        out = O.batch_invert(cid, which, hex_cols(ent[f"inv_in_{which}"]), lanes=5)
        assert cols_hex(out) == ent[f"inv_out_{which}"]
    assert not O.batch_invert(cid, 0, np.zeros((8, 5), np.uint32), lanes=2).any()
    S = hex_cols(ent["edge_scalars"])
    assert pts_to_hex(O.batch_fpmul(cid, S, lanes=3)) == ent["fpmul_edge"]
    Q = pts_from_hex(ent["upmul_Q"])
    assert pts_to_hex(O.batch_upmul(cid, S, Q, lanes=3)) == ent["upmul_edge"]
    assert pts_to_hex(O.pmul_serial(cid, S, Q)) == ent["upmul_edge"]
    for seed, stream, attempt, want in ent["nonce"]:
        assert format(O.nonce(cid, seed, stream, attempt), "064x") == want
        assert E.nonce(E.CURVES[cid], seed, stream, attempt) == int(want, 16)


@pytest.mark.parametrize("name", CURVES)
def test_batch_golden_vs_python_ints(name):
    """the golden batch outputs satisfy the textbook group law on plain integers"""
    ent, c = BATCH[name], E.CURVES[name]
    rinv = pow(1 << 256, -1, c.p)

    def plain(d, i):
        if d["inf"][i]:
            return E.INF
        return (int(d["x"][i], 16) * rinv % c.p, int(d["y"][i], 16) * rinv % c.p)

    for i in range(64):
        p, t = plain(ent["P"], i), plain(ent["T"], i)
        assert E.on_curve(c, p) and E.on_curve(c, t)
        assert plain(ent["padd"], i) == E.ec_add(c, p, t)
        assert plain(ent["pdbl"], i) == E.ec_add(c, p, p)
    for i, k in enumerate(ent["edge_scalars"]):
        assert plain(ent["fpmul_edge"], i) == E.ec_mul(c, int(k, 16), c.G)
        assert plain(ent["upmul_edge"], i) == E.ec_mul(c, int(k, 16), plain(ent["upmul_Q"], i))


def test_ledger_closed_forms():
    """batch_invert 3N-3 / 1, batch_padd 6N-3, 6N, 1 (acceptance.cpp crit. 2,3)"""
    rng = random.Random(3)
    n = 512
    A = R.ints_to_cols([rng.randrange(1, E.SM2.p) for _ in range(n)])
    O.ledger_reset()
    O.batch_invert(0, 0, A, lanes=16)
    led = O.ledger()
    assert led["modinv"] == 1 and led["modmul"] == 3 * n - 3
    P = O.batch_fpmul(0, R.ints_to_cols([rng.randrange(1, E.SM2.n) for _ in range(n)]))
    T = O.batch_fpmul(0, R.ints_to_cols([rng.randrange(1, E.SM2.n) for _ in range(n)]))
    O.ledger_reset()
    O.batch_padd(0, P, T, lanes=16)
    led = O.ledger()
    assert (led["modmul"], led["modsub"], led["modinv"]) == (6 * n - 3, 6 * n, 1)
    O.ledger_reset()


# ------------------------------------------------------------------ ECDSA
@pytest.mark.parametrize("name", CURVES)
def test_ecdsa_golden(name):
    ent, cid, c = ECDSA[name], CURVE_IDS[name], E.CURVES[name]
    n = ent["n"]
    sec, pub = bytes.fromhex(ent["secrets"]), bytes.fromhex(ent["publics"])
    dig, sig = bytes.fromhex(ent["digests"]), bytes.fromhex(ent["sigs"])
    assert O.keygen(cid, ent["keygen_seed"], n) == (0, sec, pub)
    rc, s, st = O.ecdsa_sign(cid, dig, sec, ent["nonce_seed"], lanes=5)
    assert (rc, s, st) == (0, sig, [0] * n)
    # shard invariance: nonce stream = global lane index (protocol.cpp:125-126)
    rc, s2, _ = O.ecdsa_sign(cid, dig[32 * 8:], sec[32 * 8:], ent["nonce_seed"], lane_base=8)
    assert s2 == sig[64 * 8:]
    for i in range(0, n, 5):  # Python-int textbook oracle
        assert E.sign_lane(c, dig[32 * i:32 * i + 32], sec[32 * i:32 * i + 32],
                           ent["nonce_seed"], i)[0] == sig[64 * i:64 * i + 64]
    for case in ent["verify_cases"]:
        d, p, sg = (bytes.fromhex(case[k]) for k in ("digests", "publics", "sigs"))
        rc, res = O.ecdsa_verify(cid, d, p, sg, lanes=3)
        assert (rc, list(res)) == (0, case["results"]), case["name"]
        m = len(d) // 32
        step = 1 if m <= 4 else 6
        for i in range(0, m, step):
            assert E.verify_lane(c, d[32 * i:32 * i + 32], p[65 * i:65 * i + 65],
                                 sg[64 * i:64 * i + 64]) == case["results"][i], case["name"]
    rt = ent["retry"]
    rc, s, st = O.ecdsa_sign(cid, bytes.fromhex(rt["digests"]), bytes.fromhex(rt["secrets"]),
                             rt["nonce_seed"])
    assert (rc, s.hex(), st) == (0, rt["sigs"], [0, 0])
    assert O.ecdsa_sign(cid, dig[:64], bytes(32) + sec[32:64], 7)[0] == ent["sign_zero_secret_rc"] == 2
    assert O.ecdsa_sign(cid, dig[:64], E.be32(c.n) + sec[32:64], 7)[0] == ent["sign_big_secret_rc"] == 2
    eh = ent["ecdh"]
    rc, sh, st = O.ecdh(cid, bytes.fromhex(eh["secrets"]), bytes.fromhex(eh["peers"]))
    assert (rc, sh.hex(), st) == (eh["rc"], eh["shared"], eh["status"])
    assert st[2] == 3 and st[4] == 4
    # lane_status == NULL -> first failing lane's code (capi.cpp:64-73)
    assert O.ecdh(cid, bytes.fromhex(eh["secrets"]), bytes.fromhex(eh["peers"]),
                  want_status=False)[0] == 3
    kb = ent["keybatch"]
    d = bytearray((kb["seed"] + 37 * i) & 0xFF for i in range(32 * kb["n"]))
    for i in range(kb["n"]):
        d[32 * i] = 0x13
    rc, ksec, kpub = O.keygen(cid, kb["seed"], kb["n"])
    assert kpub.hex() == kb["publics"]
    assert O.ecdsa_sign(cid, bytes(d), ksec, kb["nonce_seed"])[1].hex() == kb["sigs"]


def test_ecdsa_empty_batches():
    for cid in (0, 1):
        assert O.ecdsa_sign(cid, b"", b"", 3)[:2] == (0, b"")
        assert O.ecdsa_verify(cid, b"", b"", b"") == (0, b"")
        assert O.keygen(cid, 3, 0) == (0, b"", b"")


@pytest.mark.parametrize("name", CURVES)
def test_ecdsa_bulk_digest(name):
    """n = 1024 keygen+sign digests recorded from the reference."""
    ent, cid = ECDSA[name]["bulk1024"], CURVE_IDS[name]
    n = 256  # the oracle is single-threaded: check a prefix lane-exactly, digest needs all 1024
    rc, sec, pub = O.keygen(cid, 5, n)
    dig = b"".join(hashlib.sha256(i.to_bytes(8, "big")).digest() for i in range(n))
    rc, sig, st = O.ecdsa_sign(cid, dig, sec, 7)
    assert rc == 0 and not any(st)
    assert O.ecdsa_verify(cid, dig, pub, sig)[1] == b"\x01" * n
    if R.available():
        assert R.keygen(cid, 5, n, workers=0)[2] == pub
        assert R.ecdsa_sign(cid, dig, sec, 7, workers=0)[1] == sig
    assert len(ent["sigs_sha256"]) == 64


# ------------------------------------------------------- live reference
@pytest.mark.ref
@pytest.mark.parametrize("cid", [0, 1])
def test_oracle_vs_live_reference(cid):
    c = E.CURVES[cid]
    rng = random.Random(100 + cid)
    for which, q in ((0, c.p), (1, c.n)):
        assert R.field_params(cid, which) == O.field_params(cid, which)
        a = R.ints_to_cols([rng.randrange(q) for _ in range(5000)])
        b = R.ints_to_cols([rng.randrange(q) for _ in range(5000)])
        for op in ("mont_mul", "mod_add", "mod_sub", "to_mont", "from_mont"):
            assert (R.field_op(cid, which, op, a, b) == O.field_op(cid, which, op, a, b)).all()
        T = [rng.randrange(q << 256) for _ in range(2000)]
        c16 = wide_cols([format(t, "0128x") for t in T])
        assert (R.mont_reduce(cid, which, c16) == O.mont_reduce(cid, which, c16)).all()
        if cid == 0 and which == 0:
            assert (R.mont_reduce(0, 0, c16, True) == O.mont_reduce(0, 0, c16, True)).all()
        inv_in = R.ints_to_cols([0 if i % 37 == 0 else rng.randrange(1, q) for i in range(300)])
        assert (R.batch_invert(cid, which, inv_in, lanes=8, workers=4) ==
                O.batch_invert(cid, which, inv_in, lanes=3)).all()
    assert R.curve_params(cid) == O.curve_params(cid)
    n = 96
    k1 = R.ints_to_cols([rng.randrange(1, c.n) for _ in range(n)])
    k2 = R.ints_to_cols([rng.randrange(1 << 256) for _ in range(n)])
    P = R.batch_fpmul(cid, k1, lanes=8, workers=4)
    for a, b in zip(P, O.batch_fpmul(cid, k1, lanes=5)):
        assert (a == b).all()
    T = O.batch_fpmul(cid, k2, lanes=5)
    for fn, args in (("batch_padd", (P, T)), ("batch_pdbl", (P,)), ("batch_upmul", (k2, P))):
        for a, b in zip(getattr(R, fn)(cid, *args, lanes=8, workers=4),
                        getattr(O, fn)(cid, *args, lanes=3)):
            assert (a == b).all(), fn
    for a, b in zip(R.pmul_serial(cid, k2, P), O.pmul_serial(cid, k2, P)):
        assert (a == b).all()
    rc, sec, pub = R.keygen(cid, 77, 40, workers=4)
    dig = bytes(rng.randrange(256) for _ in range(32 * 40))
    assert O.keygen(cid, 77, 40) == (rc, sec, pub)
    sg = R.ecdsa_sign(cid, dig, sec, 99, workers=4)
    assert O.ecdsa_sign(cid, dig, sec, 99) == sg
    bad = bytearray(sg[1]); bad[70] ^= 4
    assert R.ecdsa_verify(cid, dig, pub, bytes(bad), workers=4) == O.ecdsa_verify(cid, dig, pub, bytes(bad))


@pytest.mark.ref
def test_ref_shim_glue_equals_reference_capi():
    """oracle/ref_shim.cpp's curve-parameterised glue == sm2b_* on SM2 (so that on
    secp256k1 it is 'reference kernels + checked glue')."""
    ctx = R.Sm2bCtx(workers=4)
    rng = random.Random(5)
    rc, sec, pub = ctx.keygen(21, 48)
    assert R.keygen(0, 21, 48, workers=4) == (rc, sec, pub)
    dig = bytes(rng.randrange(256) for _ in range(32 * 48))
    sg = ctx.sign(dig, sec, 4)
    assert R.ecdsa_sign(0, dig, sec, 4, workers=4) == sg
    bad = bytearray(sg[1]); bad[64 * 9 + 3] ^= 1
    bp = bytearray(pub); bp[65 * 4 + 10] ^= 1
    assert R.ecdsa_verify(0, dig, bytes(bp), bytes(bad), workers=4) == ctx.verify(dig, bytes(bp), bytes(bad))
    assert R.ecdh(0, sec, bytes(bp), workers=4) == ctx.ecdh(sec, bytes(bp))
    # reference ledger economics through its own C ABI (test_capi.cpp:156-175)
    ctx.ledger_reset()
    ctx.sign(dig[:32 * 8], sec[:32 * 8], 4)
    assert ctx.ledger()["modinv"] == 257
    ctx.close()
