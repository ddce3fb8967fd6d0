"""Runtime moduli and user curves (gecc_*_rt): FieldParams::make on the host (CPU test), the
field layer and the batched affine kernels on moduli / curves that are NOT compiled into the
library (GPU tests), against Python integers and against the compiled-in paths / the oracle.

Reference behaviour: FieldParams::make(q) (proj/src/field.cpp:159-179: odd q only, R and R^2 by
modular doublings), mont_mul / mod_add / mod_sub / inversion on a generic q (field.cpp:194-246,
proj/tests/test_field.cpp:172-201 uses a second modulus the same way), batch_invert / batch_padd /
batch_pdbl taking the field / curve as an argument (batch_invert.hpp:61, batch_point.hpp:47-60).
"""
import random

import numpy as np
import pytest

import paper_2501_03245_b200 as gecc
from oracle import coracle as O
from oracle import pyec as E

R = 1 << 256
P256 = 2**256 - 2**224 + 2**192 + 2**96 - 1           # NIST P-256 base field: a user curve, a = -3
P256_B = 0x5AC635D8AA3A93E7B3EBBD55769886BC651D06B0CC53B0F63BCE3C3E27D2604B
P256_G = (0x6B17D1F2E12C4247F8BCE6E563A440F277037D812DEB33A0F4A13945D898C296,
          0x4FE342E2FE1A7F9B8EE7EB4A7C0F9E162BCE33576B315ECECBB6406837BF51F5)
MODULI = [P256, 2**255 - 19, E.SECP256K1.n, E.SM2.p, 65537, (1 << 200) + 235, 3]  # all prime, all odd


def test_field_params_make_matches_python_ints():
    for q in MODULI:
        prm = gecc.field_params_make(q)
        assert gecc.field_params_get(prm, 0) == q
        assert gecc.field_params_get(prm, 1) == R % q
        assert gecc.field_params_get(prm, 2) == R * R % q
        assert gecc.field_params_get(prm, 3) == R * R * R % q
    for bad in (0, 1, 2, 1 << 255, E.SM2.p - 1):  # "modulus must be odd" (field.cpp:160); 1 is no field
        with pytest.raises(ValueError):
            gecc.field_params_make(bad)
    # the reference's own constants for the compiled-in fields (oracle = restated field.cpp)
    fp = O.field_params(0, 0)
    prm = gecc.field_params_make(fp["q"])
    assert gecc.field_params_get(prm, 1) == fp["r"] and gecc.field_params_get(prm, 2) == fp["r2"]


@pytest.fixture(scope="module")
def ctx():
    c = gecc.Context(gecc.SECP256K1)
    yield c
    c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("q", MODULI, ids=lambda q: f"q{q.bit_length()}")
def test_runtime_field_ops_vs_python_ints(ctx, q):
    rng = random.Random(q & 0xFFFF)
    prm = gecc.field_params_make(q)
    rinv = pow(R, -1, q)
    a = [0, 1 % q, q - 1, (q - 2) % q, (q + 1) // 2] + [rng.randrange(q) for _ in range(2000)]
    b = list(reversed(a))
    A, B = gecc.cols_from_ints(a), gecc.cols_from_ints(b)
    ints = gecc.ints_from_cols
    assert ints(ctx.field_op_rt(prm, "mont_mul", A, B)) == [x * y * rinv % q for x, y in zip(a, b)]
    assert ints(ctx.field_op_rt(prm, "mod_add", A, B)) == [(x + y) % q for x, y in zip(a, b)]
    assert ints(ctx.field_op_rt(prm, "mod_sub", A, B)) == [(x - y) % q for x, y in zip(a, b)]
    assert ints(ctx.field_op_rt(prm, "to_mont", A)) == [x * R % q for x in a]
    assert ints(ctx.field_op_rt(prm, "from_mont", A)) == [x * rinv % q for x in a]
    want_inv = [pow(x * rinv % q, -1, q) * R % q if x else 0 for x in a]
    assert ints(ctx.field_op_rt(prm, "mod_inv", A)) == want_inv
    assert ints(ctx.field_op_rt(prm, "mod_inv_fermat", gecc.cols_from_ints(a[:64]))) == want_inv[:64]
    assert ints(ctx.batch_invert_rt(prm, A)) == want_inv   # zero -> zero, neighbours unaffected


@pytest.mark.gpu
@pytest.mark.parametrize("cid", [0, 1])
def test_runtime_field_equals_compiled_field_and_oracle(ctx, cid):
    """the same modulus through the runtime route and through the compiled-in one (both fields)"""
    with gecc.Context(cid) as c:
        for which in (0, 1):
            q = O.field_params(cid, which)["q"]
            prm = gecc.field_params_make(q)
            rng = random.Random(5 + which)
            A = gecc.cols_from_ints([rng.randrange(q) for _ in range(3000)])
            B = gecc.cols_from_ints([rng.randrange(q) for _ in range(3000)])
            for op in ("mont_mul", "mod_add", "mod_sub", "to_mont", "from_mont"):
                got = c.field_op_rt(prm, op, A, B)
                assert (got == c.field_op(which, op, A, B)).all(), op
                assert (got == O.field_op(cid, which, op, A, B)).all(), op
            assert (c.batch_invert_rt(prm, A) == O.batch_invert(cid, which, A)).all()


def _mont_points(q, pts):
    xs = gecc.cols_from_ints([0 if p is None else p[0] * R % q for p in pts])
    ys = gecc.cols_from_ints([0 if p is None else p[1] * R % q for p in pts])
    return xs, ys, np.array([1 if p is None else 0 for p in pts], np.uint8)


def _plain_points(q, P):
    rinv = pow(R, -1, q)
    xs, ys = gecc.ints_from_cols(P[0]), gecc.ints_from_cols(P[1])
    return [None if P[2][i] else (xs[i] * rinv % q, ys[i] * rinv % q) for i in range(len(xs))]


@pytest.mark.gpu
def test_user_curve_p256_padd_pdbl_vs_python_ints(ctx):
    """NIST P-256 is not compiled into the library: batch_padd / batch_pdbl on CurveParams given at
    run time, with the exceptional-lane set of proj/tests/test_batch_point.cpp:70-100 (equal points,
    opposite points, infinity on either side / both sides) spliced in."""
    c = E.Curve("p256", 9, P256, P256 - 3, P256_B, 0xFFFFFFFF00000000FFFFFFFFFFFFFFFFBCE6FAADA7179E84F3B9CAC2FC632551, *P256_G)
    assert E.on_curve(c, c.G)
    rng = random.Random(256)
    n = 700
    base = [E.ec_mul(c, rng.randrange(1, 1 << 64), c.G) for _ in range(40)]
    P = [base[rng.randrange(40)] for _ in range(n)]
    T = [base[rng.randrange(40)] for _ in range(n)]          # 40 distinct points: equal pairs occur on their own
    P[3], T[3] = base[0], base[0]                             # doubling lane
    P[7], T[7] = base[1], E.ec_neg(c, base[1])                # inverse pair
    P[11], T[11] = None, base[2]
    P[19], T[19] = base[3], None
    P[23], T[23] = None, None
    prm = gecc.field_params_make(P256)
    a_mont = gecc.cols_from_ints([(P256 - 3) * R % P256])[:, 0].copy()
    got = _plain_points(P256, ctx.batch_padd_rt(prm, a_mont, _mont_points(P256, P), _mont_points(P256, T)))
    assert got == [E.ec_add(c, p, t) for p, t in zip(P, T)]
    got = _plain_points(P256, ctx.batch_pdbl_rt(prm, a_mont, _mont_points(P256, P)))
    assert got == [E.ec_add(c, p, p) for p in P]
    # infinity results carry zero coordinates (batch_point.cpp:41-47)
    S = ctx.batch_padd_rt(prm, a_mont, _mont_points(P256, P), _mont_points(P256, T))
    assert S[2][7] == 1 and S[2][23] == 1 and not S[0][:, 7].any() and not S[1][:, 23].any()


@pytest.mark.gpu
@pytest.mark.parametrize("cid", [0, 1])
def test_runtime_curve_equals_compiled_curve(cid):
    """SM2 / secp256k1 given as runtime CurveParams: bit-identical to the compiled-in batch kernels
    and to the oracle (restated batch_point.cpp), exceptional lanes included."""
    c = E.CURVES[cid]
    with gecc.Context(cid) as ctx:
        n = 1500
        ks = gecc.cols_from_ints([random.Random(cid).randrange(1, c.n) for _ in range(n)])
        ts = gecc.cols_from_ints([random.Random(cid + 9).randrange(1, c.n) for _ in range(n)])
        P, T = [list(x) for x in (ctx.batch_fpmul(ks), ctx.batch_fpmul(ts))]
        for X in (P, T):
            X[0], X[1], X[2] = X[0].copy(), X[1].copy(), X[2].copy()
        T[0][:, 5], T[1][:, 5] = P[0][:, 5], P[1][:, 5]                      # equal
        T[0][:, 9] = P[0][:, 9]
        T[1][:, 9] = gecc.cols_from_ints([(c.p - v) % c.p for v in gecc.ints_from_cols(P[1][:, 9:10])])[:, 0]  # opposite
        P[2][13] = 1; P[0][:, 13] = 0; P[1][:, 13] = 0
        T[2][17] = 1; T[0][:, 17] = 0; T[1][:, 17] = 0
        prm = gecc.field_params_make(c.p)
        a_mont = gecc.cols_from_ints([c.a * R % c.p])[:, 0].copy()
        got = ctx.batch_padd_rt(prm, a_mont, tuple(P), tuple(T))
        want = ctx.batch_padd(tuple(P), tuple(T))
        ora = O.batch_padd(cid, tuple(P), tuple(T))
        for g, w, o in zip(got, want, ora):
            assert (g == w).all() and (g == np.asarray(o)).all()
        got = ctx.batch_pdbl_rt(prm, a_mont, tuple(P))
        for g, w in zip(got, ctx.batch_pdbl(tuple(P))):
            assert (g == w).all()


@pytest.mark.gpu
def test_runtime_entry_points_reject_bad_arguments(ctx):
    prm = gecc.field_params_make(P256)
    A = gecc.cols_from_ints([1, 2, 3])
    l = gecc.lib()
    out = np.zeros((8, 3), np.uint32)
    blank = np.zeros(64, np.uint32)  # a parameter block that gecc_field_params_make did not fill
    assert l.gecc_field_op_rt(ctx.h, blank.ctypes.data, 0, 3, A.ctypes.data, A.ctypes.data, out.ctypes.data) == 1
    assert l.gecc_field_op_rt(ctx.h, prm.ctypes.data, 0, 3, A.ctypes.data, None, out.ctypes.data) == 1   # binary op without b
    assert l.gecc_field_op_rt(ctx.h, prm.ctypes.data, 7, 3, A.ctypes.data, A.ctypes.data, out.ctypes.data) == 1  # opcode outside the runtime set
    assert l.gecc_batch_invert_rt(ctx.h, prm.ctypes.data, 0, None, None) == 0                              # empty batch
