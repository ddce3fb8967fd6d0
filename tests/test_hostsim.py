"""CPU tests of the *product's* device code, compiled for the host (tests/hostsim).

The authoring container has no GPU, so the __host__ __device__ limb, curve and
ECDSA-lane code under paper_2501_03245_b200/csrc is built with g++ (the PTX carry
flag is emulated, and the emulation aborts on add/sub flag-family mixing, which is
wrong on hardware) and checked against the oracle and the golden vectors here.
The same code paths are then re-checked on the B200 by the `gpu` tests.
"""
import random

import numpy as np
import pytest

from oracle import coracle as O
from oracle import pyec as E
from tests.hostsim import hostsim as H
from tests.util import CURVE_IDS, cols_hex, golden, hex_cols, pts_from_hex, pts_to_hex, wide_cols

FIELD, BATCH, ECDSA = golden("field"), golden("batch"), golden("ecdsa")
CURVES = ["sm2", "secp256k1"]


@pytest.mark.parametrize("key", [k for k in FIELD if not k.startswith("_")])
def test_hostsim_field_golden(key):
    ent = FIELD[key]
    cid = CURVE_IDS[key.split(".")[0]]
    which = 0 if key.endswith(".p") else 1
    A, B = hex_cols(ent["a"]), hex_cols(ent["b"])
    for op in ("mont_mul", "mod_add", "mod_sub", "to_mont", "from_mont", "mod_inv"):
        assert cols_hex(H.field_op(cid, which, op, A, B)) == ent[op], op


@pytest.mark.parametrize("key", [k for k in FIELD if not k.startswith("_")])
def test_hostsim_reduce_edges(key):
    """512-bit reduce edge values of test_field.cpp:136-164 through every reduction route
    (secp256k1 word-serial, SM2 add/sub-only, generic two-product REDC)."""
    ent = FIELD[key]
    cid = CURVE_IDS[key.split(".")[0]]
    which = 0 if key.endswith(".p") else 1
    q = int(ent["q"], 16)
    rng = random.Random(77)
    extra = [format(rng.randrange(q << 256), "0128x") for _ in range(3000)]
    c16 = wide_cols(ent["reduce_in"] + extra)
    got = cols_hex(H.redc(cid, which, c16))
    assert got[:len(ent["reduce_in"])] == ent["reduce_generic"]
    assert got == cols_hex(O.mont_reduce(cid, which, c16, False))


def test_hostsim_inverse_and_glv():
    """safegcd inversion vs the oracle's Fermat value; GLV split k = k1 + k2 lambda mod n."""
    rng = random.Random(8)
    for cid in (0, 1):
        for which in (0, 1):
            q = O.field_params(cid, which)["q"]
            vals = [0, 1, 2, q - 1, q - 2, (q + 1) // 2, (1 << 128) - 1] + [rng.randrange(q) for _ in range(1500)]
            a = O.ints_to_cols(vals)
            assert (H.field_op(cid, which, "inv_safegcd", a) == O.field_op(cid, which, "mod_inv", a)).all()
            plain = O.cols_to_ints(H.field_op(cid, which, "inv_plain", a))
            assert all(g == (pow(v, -1, q) if v else 0) for g, v in zip(plain, vals))
            # the variable-time form (block totals of Montgomery's trick) gives the same residues
            assert (H.field_op(cid, which, "inv_var", a) == O.field_op(cid, which, "mod_inv", a)).all()
            assert O.cols_to_ints(H.field_op(cid, which, "inv_var_plain", a)) == plain
            # the software-pipelined schedule of the same rounds, with and without the early exit
            assert O.cols_to_ints(H.field_op(cid, which, "inv_sched_plain", a)) == plain
            assert O.cols_to_ints(H.field_op(cid, which, "inv_sched_exit_plain", a)) == plain
    n = E.SECP256K1.n
    lam = 0x5363AD4CC05C30E0A5261C028812645A122E22EA20816678DF02967C1B23BD72
    ks = [0, 1, 2, n - 1, n - 2, lam, n - lam, (n - 1) // 2, 1 << 255] + [rng.randrange(n) for _ in range(5000)]
    m1, m2, sg = H.glv_split(O.ints_to_cols(ks))
    a, b = O.cols_to_ints(m1), O.cols_to_ints(m2)
    for i, k in enumerate(ks):
        k1 = -a[i] if sg[2 * i] else a[i]
        k2 = -b[i] if sg[2 * i + 1] else b[i]
        assert (k1 + k2 * lam - k) % n == 0 and a[i] < 1 << 129 and b[i] < 1 << 129


@pytest.mark.parametrize("cid", [0, 1])
@pytest.mark.parametrize("which", [0, 1])
def test_hostsim_field_random(cid, which):
    q = O.field_params(cid, which)["q"]
    rng = random.Random(50 + 2 * cid + which)
    edge = [0, 1, 2, q - 1, q - 2, (1 << 255) % q, (1 << 224) - 1, q >> 1, 0xFFFFFFFF, ((q - 1) ^ 0xFFFFFFFF) % q]
    a = O.ints_to_cols(edge + [rng.randrange(q) for _ in range(4000)])
    b = O.ints_to_cols(edge[::-1] + [rng.randrange(q) for _ in range(4000)])
    for op in ("mont_mul", "mod_add", "mod_sub", "to_mont", "from_mont"):
        assert (H.field_op(cid, which, op, a, b) == O.field_op(cid, which, op, a, b)).all(), op
    assert (H.field_op(cid, which, "sqr", a) == O.field_op(cid, which, "mont_mul", a, a)).all()


@pytest.mark.parametrize("name", CURVES)
def test_hostsim_point_mul_golden(name):
    ent, cid = BATCH[name], CURVE_IDS[name]
    S = hex_cols(ent["edge_scalars"])
    assert pts_to_hex(H.batch_fpmul(cid, S)) == ent["fpmul_edge"]
    Q = pts_from_hex(ent["upmul_Q"])
    assert pts_to_hex(H.batch_upmul(cid, S, Q)) == ent["upmul_edge"]
    rng = random.Random(9)
    k = O.ints_to_cols([rng.randrange(1 << 256) for _ in range(24)])
    P = O.batch_fpmul(cid, k)
    for a, b in zip(H.batch_fpmul(cid, k), P):
        assert (a == b).all()
    k2 = O.ints_to_cols([rng.randrange(1 << 256) for _ in range(24)])
    for a, b in zip(H.batch_upmul(cid, k2, P), O.pmul_serial(cid, k2, P)):
        assert (a == b).all()


@pytest.mark.parametrize("name", CURVES)
def test_hostsim_ecdsa_golden(name):
    ent, cid = ECDSA[name], CURVE_IDS[name]
    n = ent["n"]
    sec, pub = bytes.fromhex(ent["secrets"]), bytes.fromhex(ent["publics"])
    dig, sig = bytes.fromhex(ent["digests"]), bytes.fromhex(ent["sigs"])
    assert H.keygen(cid, ent["keygen_seed"], n) == (sec, pub)
    assert H.sign(cid, dig, sec, ent["nonce_seed"]) == (sig, [0] * n)
    assert H.sign(cid, dig[32 * 8:], sec[32 * 8:], ent["nonce_seed"], lane_base=8)[0] == sig[64 * 8:]
    for case in ent["verify_cases"]:
        d, p, sg = (bytes.fromhex(case[k]) for k in ("digests", "publics", "sigs"))
        assert list(H.verify(cid, d, p, sg)) == case["results"], case["name"]
    rt = ent["retry"]
    s, st = H.sign(cid, bytes.fromhex(rt["digests"]), bytes.fromhex(rt["secrets"]), rt["nonce_seed"])
    assert (s.hex(), st) == (rt["sigs"], [0, 0])


def test_hostsim_lazy_secp_field():
    """The lazy plain secp256k1 field of the fused ECDSA kernels: weakly reduced 256-bit values,
    including NON-canonical inputs (q, q+1, 2^256-1 ...), against Python integers mod q."""
    p = E.SECP256K1.p
    rng = random.Random(11)
    special = [0, 1, p - 1, p, p + 1, 2**256 - 1, 2**256 - 2, p + 977, 2**255, 2**256 - 2**32, 2**256 - 977, 5]
    a = special + [rng.randrange(1 << 256) for _ in range(5000)]
    b = special[::-1] + [rng.randrange(1 << 256) for _ in range(5000)]
    A, B = O.ints_to_cols(a), O.ints_to_cols(b)
    for op, fn in (("mont_mul", lambda x, y: x * y), ("mod_add", lambda x, y: x + y),
                   ("mod_sub", lambda x, y: x - y), ("sqr", lambda x, y: x * x)):
        got = O.cols_to_ints(H.field_op(1, 0, op, A, B, field_id=H.SECP_LAZY_FIELD))
        assert all(g % p == fn(x, y) % p for g, x, y in zip(got, a, b)), op
    canon = O.cols_to_ints(H.field_op(1, 0, "from_mont", A, field_id=H.SECP_LAZY_FIELD))
    assert canon == [x % p for x in a]
    # doubling / x8 by funnel shifts: edge values whose shifted-out bits and low limbs hit the
    # rare carry branches, on the lazy field and (as add chains) on the Montgomery field
    sh = edge_vals = special + [2**256 - 2**32, 2**255 + 2**64 - 1, (7 << 253) | (2**64 - 1), (7 << 253) | (2**64 - 978),
                                2**256 - 2**61, (1 << 253) - 1, 0xFFFFFFFF << 32, (0xE0000000 << 224) | (2**256 - 1) >> 35]
    sh = sh + [rng.randrange(1 << 256) for _ in range(2000)]
    SH = O.ints_to_cols(sh)
    for op, kk in (("dbl", 2), ("mul8", 8)):
        got = O.cols_to_ints(H.field_op(1, 0, op, SH, field_id=H.SECP_LAZY_FIELD))
        assert all(g % p == kk * x % p and g < (1 << 256) for g, x in zip(got, sh)), op
        canon_in = O.ints_to_cols([x % p for x in sh])
        got = O.cols_to_ints(H.field_op(1, 0, op, canon_in))
        assert got == [kk * x % p for x in sh], op
    # every pair of edge values: drives the rare branches of the folds (carry / borrow rippling
    # out of limb 1, and the second wrap at a >= 2^256 - c or d < c)
    edge = special + [2**64 - 1, 2**64, 2**64 - 977, 2**256 - 2**64, 2**256 - 2**64 + 1, 977, 976, 2**32 + 977,
                      2**32 + 976, 2**256 - 2**32 - 978, (1 << 256) - (1 << 33), 2**96 - 1]
    xa = [x for x in edge for _ in edge]
    xb = [y for _ in edge for y in edge]
    XA, XB = O.ints_to_cols(xa), O.ints_to_cols(xb)
    for op, fn in (("mont_mul", lambda x, y: x * y), ("mod_add", lambda x, y: x + y), ("mod_sub", lambda x, y: x - y)):
        got = O.cols_to_ints(H.field_op(1, 0, op, XA, XB, field_id=H.SECP_LAZY_FIELD))
        assert all(g % p == fn(x, y) % p for g, x, y in zip(got, xa, xb)), op
    inv = O.cols_to_ints(H.field_op(1, 0, "inv_safegcd", np.ascontiguousarray(A[:, :400]), field_id=H.SECP_LAZY_FIELD))
    assert all((g * x) % p == 1 if x % p else g == 0 for g, x in zip(inv, a[:400]))
    inv = O.cols_to_ints(H.field_op(1, 0, "inv_var", np.ascontiguousarray(A[:, :400]), field_id=H.SECP_LAZY_FIELD))
    assert all((g * x) % p == 1 if x % p else g == 0 for g, x in zip(inv, a[:400]))


def test_hostsim_lazy_sm2_field():
    """The weakly reduced Montgomery SM2 field of the fused ECDSA kernels on NON-canonical inputs
    (q, q + 1, 2^256 - 1, values around c = 2^256 - q ...), against Python integers mod q; every pair
    of edge values drives the second-wrap branches of the carry / borrow folds."""
    p = E.SM2.p
    c = (1 << 256) - p
    rinv = pow(1 << 256, -1, p)
    rng = random.Random(12)
    special = [0, 1, p - 1, p, p + 1, 2**256 - 1, 2**256 - 2, c, c - 1, c + 1, 2 * c, 2**255, p - c, 2**224, 2**96 - 2**64, 5]
    a = special + [rng.randrange(1 << 256) for _ in range(5000)]
    b = special[::-1] + [rng.randrange(1 << 256) for _ in range(5000)]
    A, B = O.ints_to_cols(a), O.ints_to_cols(b)
    f = H.SM2_LAZY_FIELD
    for op, fn in (("mont_mul", lambda x, y: x * y * rinv), ("mod_add", lambda x, y: x + y),
                   ("mod_sub", lambda x, y: x - y), ("sqr", lambda x, y: x * x * rinv), ("dbl", lambda x, y: 2 * x),
                   ("mul8", lambda x, y: 8 * x)):
        got = O.cols_to_ints(H.field_op(0, 0, op, A, B, field_id=f))
        assert all(g % p == fn(x, y) % p and g < (1 << 256) for g, x, y in zip(got, a, b)), op
    assert O.cols_to_ints(H.field_op(0, 0, "from_mont", A, field_id=f)) == [x * rinv % p for x in a]
    assert all(g % p == x * (1 << 256) % p for g, x in zip(O.cols_to_ints(H.field_op(0, 0, "to_mont", A, field_id=f)), a))
    edge = special + [2**64 - 1, 2**64, 2**256 - 2**64, 2**256 - c, 2**256 - c - 1, 2**256 - c + 1, 2**96, 2**224 - 1, (1 << 256) - (1 << 33)]
    xa = [x for x in edge for _ in edge]
    xb = [y for _ in edge for y in edge]
    XA, XB = O.ints_to_cols(xa), O.ints_to_cols(xb)
    for op, fn in (("mont_mul", lambda x, y: x * y * rinv), ("mod_add", lambda x, y: x + y), ("mod_sub", lambda x, y: x - y)):
        got = O.cols_to_ints(H.field_op(0, 0, op, XA, XB, field_id=f))
        assert all(g % p == fn(x, y) % p for g, x, y in zip(got, xa, xb)), op
    # canonical inputs: the lazy field's values equal the canonical field's mod q
    ca = O.ints_to_cols([x % p for x in a[:2000]])
    cb = O.ints_to_cols([x % p for x in b[:2000]])
    want = O.cols_to_ints(O.field_op(0, 0, "mont_mul", ca, cb))
    assert [g % p for g in O.cols_to_ints(H.field_op(0, 0, "mont_mul", ca, cb, field_id=f))] == want
    R = 1 << 256
    for op in ("inv_safegcd", "inv_var"):
        inv = O.cols_to_ints(H.field_op(0, 0, op, np.ascontiguousarray(A[:, :400]), field_id=f))
        assert all((g * x * rinv * rinv) % p == 1 if x % p else g % p == 0 for g, x in zip(inv, a[:400])), op


@pytest.mark.parametrize("curve_name,cid", [("secp256k1", H.SECP_LAZY_CURVE), ("sm2", H.SM2_LAZY_CURVE)])
def test_hostsim_lazy_curve_ecdsa_golden(curve_name, cid):
    ent = ECDSA[curve_name]
    n = ent["n"]
    sec, pub = bytes.fromhex(ent["secrets"]), bytes.fromhex(ent["publics"])
    dig, sig = bytes.fromhex(ent["digests"]), bytes.fromhex(ent["sigs"])
    assert H.keygen(cid, ent["keygen_seed"], n) == (sec, pub)
    assert H.sign(cid, dig, sec, ent["nonce_seed"]) == (sig, [0] * n)
    for case in ent["verify_cases"]:
        d, p, sg = (bytes.fromhex(case[k]) for k in ("digests", "publics", "sigs"))
        assert list(H.verify(cid, d, p, sg)) == case["results"], case["name"]
    rt = ent["retry"]
    assert H.sign(cid, bytes.fromhex(rt["digests"]), bytes.fromhex(rt["secrets"]), rt["nonce_seed"])[0].hex() == rt["sigs"]


@pytest.mark.parametrize("cid,hs_curve", [(0, 0), (0, 3), (1, 1), (1, 2)])
def test_hostsim_sign_group_retry(cid, hs_curve):
    """A forced s == 0 on attempt 0 INSIDE a 4-lane group (shared inversions) must retry that
    lane with a fresh nonce exactly as the reference does (test_protocol.cpp:196-228)."""
    c = E.CURVES[cid]
    rng = random.Random(99 + cid)
    n, seed, rig = 8, 13, 5
    sec = b"".join(E.be32(rng.randrange(1, c.n)) for _ in range(n))
    dig = bytearray(rng.randrange(256) for _ in range(32 * n))
    d = int.from_bytes(sec[32 * rig:32 * rig + 32], "big")
    k0 = E.nonce(c, seed, rig, 0)
    r0 = E.ec_mul(c, k0, c.G)[0] % c.n
    dig[32 * rig:32 * rig + 32] = E.be32((-r0 * d) % c.n)      # e + r d == 0  ->  s == 0
    want = O.ecdsa_sign(cid, bytes(dig), sec, seed)
    assert want[2] == [0] * n
    k1 = E.nonce(c, seed, rig, 1)
    assert want[1][64 * rig:64 * rig + 32] == E.be32(E.ec_mul(c, k1, c.G)[0] % c.n)  # really retried
    assert H.sign(hs_curve, bytes(dig), sec, seed) == (want[1], want[2])


@pytest.mark.parametrize("cid,hs_curve", [(0, 0), (1, 1), (1, 2)])
def test_hostsim_uniform_mode_equals_fast(cid, hs_curve):
    """GECC_SECRET_UNIFORM (constant-structure k*G / k*P: every window adds, entries by select,
    SPEC.md 'constant structure', batch_point.cpp:319-333,420) gives the same bytes as the fast
    path and as the oracle -- edge scalars {0, 1, 2^77, n-1, all-ones}, zero-digit-heavy scalars,
    random scalars, keygen and sign."""
    c = E.CURVES[cid]
    rng = random.Random(31 + hs_curve)
    W = H.lib().hs_window_bits()
    sparse = [1 << (W * j) for j in range(0, 256 // W, 7)] + [(1 << 255) | 1, c.n - (1 << 200), (1 << (W * 5)) - 1]
    ks = [0, 1, 2, 1 << 77, c.n - 1, c.n - 2, (1 << 256) - 1, c.n, c.n + 1] + sparse + [rng.randrange(1 << 256) for _ in range(40)]
    k = O.ints_to_cols(ks)
    try:
        H.set_uniform(False)
        fast_f = H.batch_fpmul(hs_curve, k)
        if hs_curve != 2:   # column-buffer checks need the Montgomery-form curve
            P = O.batch_fpmul(cid, O.ints_to_cols([rng.randrange(1, c.n) for _ in ks]))
            fast_u = H.batch_upmul(hs_curve, k, P)
        H.set_uniform(True)
        uni_f = H.batch_fpmul(hs_curve, k)
        for a, b in zip(fast_f, uni_f):
            assert (a == b).all()
        if hs_curve != 2:
            want = O.batch_fpmul(cid, k)
            for a, b in zip(uni_f, want):
                assert (a == b).all()
            uni_u = H.batch_upmul(hs_curve, k, P)
            for a, b, w in zip(fast_u, uni_u, O.pmul_serial(cid, k, P)):
                assert (a == b).all() and (a == w).all()
        ent = ECDSA["secp256k1" if cid == 1 else "sm2"]
        n = ent["n"]
        sec, pub = bytes.fromhex(ent["secrets"]), bytes.fromhex(ent["publics"])
        dig, sig = bytes.fromhex(ent["digests"]), bytes.fromhex(ent["sigs"])
        assert H.keygen(hs_curve, ent["keygen_seed"], n) == (sec, pub)
        assert H.sign(hs_curve, dig, sec, ent["nonce_seed"]) == (sig, [0] * n)
    finally:
        H.set_uniform(False)


@pytest.mark.parametrize("cid,hs_curve", [(0, 0), (1, 2)])
def test_hostsim_sign_with_explicit_nonces(cid, hs_curve):
    """gecc_sign_nonces' lane: with the deterministic source's attempt-0 nonces it reproduces
    sm2b_sign; a nonce outside (0, n) and a rigged s == 0 ask for a replacement (status 5)."""
    c = E.CURVES[cid]
    rng = random.Random(5 + cid)
    n, seed = 10, 21
    sec = b"".join(E.be32(rng.randrange(1, c.n)) for _ in range(n))
    dig = bytearray(rng.randrange(256) for _ in range(32 * n))
    nonces = bytearray(b"".join(E.be32(E.nonce(c, seed, i, 0)) for i in range(n)))
    want = O.ecdsa_sign(cid, bytes(dig), sec, seed)
    assert H.sign_nonces(hs_curve, bytes(dig), sec, bytes(nonces)) == (want[1], [0] * n)
    # lane 3: nonce 0; lane 4: nonce n; lane 6: e + r d == 0 -> s == 0
    nonces[32 * 3:32 * 4] = bytes(32)
    nonces[32 * 4:32 * 5] = E.be32(c.n)
    d6 = int.from_bytes(sec[32 * 6:32 * 7], "big")
    r6 = E.ec_mul(c, E.nonce(c, seed, 6, 0), c.G)[0] % c.n
    dig[32 * 6:32 * 7] = E.be32((-r6 * d6) % c.n)
    sig, st = H.sign_nonces(hs_curve, bytes(dig), sec, bytes(nonces))
    assert st == [0, 0, 0, 5, 5, 0, 5, 0, 0, 0]
    for i in (3, 4, 6):
        assert sig[64 * i:64 * i + 64] == bytes(64)
    for i in (0, 1, 2, 5, 7, 8, 9):
        assert sig[64 * i:64 * i + 64] == want[1][64 * i:64 * i + 64]


@pytest.mark.parametrize("cid,hs_curve", [(0, 0), (0, 3), (1, 1), (1, 2)])
def test_hostsim_slot_additions_complete(cid, hs_curve):
    """jac_madd_slots / jac_mmadd_slots and the (X, Y, ZZ, ZZZ) forms of the fixed-base walk against
    jac_madd: generic pairs, Q == P (tangent), Q == -P (infinity), accumulator affine, rescaled by a
    random Z, and at infinity; each pair also with the row negated."""
    from tests.util import ints_to_cols
    c = E.CURVES[cid]
    rng = random.Random(4242 + hs_curve)
    a = [rng.randrange(1, c.n) for _ in range(12)]
    b = [rng.randrange(1, c.n) for _ in range(12)]
    for i in (1, 5):
        b[i] = a[i]            # same point
    for i in (2, 7):
        b[i] = c.n - a[i]      # inverse point
    P = H.batch_fpmul(hs_curve, ints_to_cols(a))
    Q = H.batch_fpmul(hs_curve, ints_to_cols(b))
    assert not P[2].any() and not Q[2].any()
    lam = ints_to_cols([rng.randrange(2, 1 << 250) for _ in a])
    assert H.slot_adds(hs_curve, P, Q, lam) == 0
