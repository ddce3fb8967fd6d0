"""GPU parity of the 12-limb layer (BLS12-381 and BLS12-377 G1 contexts): field kernels, batched affine
addition / doubling / inversion over 12-limb column buffers, and MSM -- against Python
integers (oracle/pyec.py).  The reference is 256-bit only, so parity is against the definition;
the same device code is also checked on the CPU by tests/test_hostsim_bls.py."""
import random

import numpy as np
import pytest

import paper_2501_03245_b200 as gecc
from oracle import pyec as E

pytestmark = pytest.mark.gpu
R12 = 1 << 384


class Env:
    """one curve: its oracle parameters, a GPU context, Montgomery conversions"""

    def __init__(self, curve, gid):
        self.B, self.ctx, self.rinv = curve, gecc.Context(gid), pow(R12, -1, curve.p)


@pytest.fixture(scope="module", params=["bls12_381", "bls12_377"])
def env(request):
    e = Env(E.CURVES[request.param], {"bls12_381": gecc.BLS12_381, "bls12_377": gecc.BLS12_377}[request.param])
    yield e
    e.ctx.close()


def cols(v, limbs=12):
    return gecc.cols_from_ints(v, limbs)


def mont_pts(B, pts):
    xs = [0 if p is None else p[0] * R12 % B.p for p in pts]
    ys = [0 if p is None else p[1] * R12 % B.p for p in pts]
    return cols(xs), cols(ys), np.array([p is None for p in pts], np.uint8)


def from_mont_pts(B, P):
    rinv = pow(R12, -1, B.p)
    xs, ys = gecc.ints_from_cols(P[0]), gecc.ints_from_cols(P[1])
    return [None if P[2][i] else (xs[i] * rinv % B.p, ys[i] * rinv % B.p) for i in range(len(xs))]


def rand_points(B, rng, n):
    """n random multiples of G, built from a few oracle points by cheap additions"""
    seeds = [E.ec_mul(B, rng.randrange(1, B.n), B.G) for _ in range(6)]
    pts, cur = [], seeds[0]
    for i in range(n):
        cur = E.ec_add(B, cur, seeds[1 + i % 5])
        pts.append(cur)
    return pts


def test_field12_kernels(env):
    B, ctx, RINV = env.B, env.ctx, env.rinv
    q = B.p
    rng = random.Random(3811)
    a = [0, 1, 2, q - 1, q - 2, (q + 1) // 2, (1 << 376) % q] + [rng.randrange(q) for _ in range(5000)]
    b = list(reversed(a))
    A, Bc = cols(a), cols(b)
    ints = gecc.ints_from_cols
    assert A.shape == (12, len(a))
    assert ints(ctx.field_op(0, "mont_mul", A, Bc)) == [x * y * RINV % q for x, y in zip(a, b)]
    assert ints(ctx.field_op(0, "mod_add", A, Bc)) == [(x + y) % q for x, y in zip(a, b)]
    assert ints(ctx.field_op(0, "mod_sub", A, Bc)) == [(x - y) % q for x, y in zip(a, b)]
    assert ints(ctx.field_op(0, "to_mont", A)) == [x * R12 % q for x in a]
    assert ints(ctx.field_op(0, "from_mont", A)) == [x * RINV % q for x in a]
    want = [pow(x * RINV % q, -1, q) * R12 % q if x else 0 for x in a]
    assert ints(ctx.field_op(0, "mod_inv", A)) == want                      # safegcd, 13 x 30-bit limbs
    assert ints(ctx.field_op(0, "mod_inv_warp", A)) == want                 # the same by a whole warp per element
    assert ints(ctx.field_op(0, "mod_inv_fermat", cols(a[:64]))) == want[:64]
    # batch inversion (Montgomery's trick, one inversion per block), zeros masked
    assert ints(ctx.batch_invert(0, A)) == want
    # the 255-bit scalar field keeps 8 limbs
    r = B.n
    s = [0, 1, r - 1] + [rng.randrange(r) for _ in range(1000)]
    rinv = pow(1 << 256, -1, r)
    S = cols(s, 8)
    assert ints(ctx.field_op(1, "mont_mul", S, S)) == [x * x * rinv % r for x in s]
    assert ints(ctx.batch_invert(1, S)) == [pow(x * rinv % r, -1, r) * (1 << 256) % r if x else 0 for x in s]


def test_batch_padd_pdbl_g1(env):
    B, ctx = env.B, env.ctx
    rng = random.Random(3812)
    n = 700  # more than one block; ragged tail
    P = rand_points(B, rng, n)
    T = list(reversed(rand_points(B, rng, n)))
    # exceptional lanes (test_batch_point.cpp:70-100): P == T, P == -T, infinities
    for i in (3, 7, 11):
        T[i] = P[i]
    for i in (19, 23):
        T[i] = (P[i][0], B.p - P[i][1])
    P[31], T[47], P[48], T[48] = None, None, None, None
    got = from_mont_pts(B, ctx.batch_padd(mont_pts(B, P), mont_pts(B, T)))
    assert got == [E.ec_add(B, a, b) for a, b in zip(P, T)]
    got = from_mont_pts(B, ctx.batch_pdbl(mont_pts(B, P)))
    assert got == [E.ec_add(B, a, a) for a in P]
    assert all(E.on_curve(B, p) for p in got)


@pytest.mark.parametrize("form", ["affine", "fused16", "fused8", "jacobian"])
def test_msm_g1(env, form):
    B, ctx = env.B, env.ctx
    gecc.set_msm_form(form)
    try:
        rng = random.Random(3813)
        for n in (1, 2, 33, 300):
            pts = rand_points(B, rng, n)
            ks = [rng.randrange(1 << 256) for _ in range(n)]
            if n == 300:  # duplicates, opposite points, zero / order / all-ones scalars, an infinity input
                for i in range(10, 40):
                    pts[i] = pts[10]
                    ks[i] = 5
                ks[0], ks[1], ks[2], ks[3] = 0, B.n, B.n - 1, (1 << 256) - 1
                pts[50] = (pts[51][0], B.p - pts[51][1])
                ks[50] = ks[51] = 77
                pts[60] = None
            want = None
            for k, p in zip(ks, pts):
                want = E.ec_add(B, want, E.ec_mul(B, k % B.n, p) if p is not None else None)
            got = from_mont_pts(B, ctx.msm(cols(ks, 8), mont_pts(B, pts)))
            assert got == [want], n
        # everything cancels / empty sum
        pts = rand_points(B, rng, 4)
        assert ctx.msm(cols([0] * 4, 8), mont_pts(B, pts))[2][0] == 1
        empty = (np.zeros((12, 0), np.uint32), np.zeros((12, 0), np.uint32), np.zeros(0, np.uint8))
        assert ctx.msm(np.zeros((8, 0), np.uint32), empty)[2][0] == 1
    finally:
        gecc.set_msm_form("auto")


def test_msm_g1_identity_2_16(env):
    B, ctx = env.B, env.ctx
    """sum_i s_i (t_i G) = (sum_i s_i t_i mod r) G at 2^16 points whose discrete logs t_i are
    known by construction (chains of batch_padd steps from oracle points, ends re-checked)."""
    rng = random.Random(3814)
    n = 1 << 16
    d = [rng.randrange(1, B.n) for _ in range(6)]
    seeds = [E.ec_mul(B, x, B.G) for x in d]
    # 256 lanes walk P <- P + D_(step mod 5) with batch_padd; every point's discrete log is known
    lanes = 256
    per = n // lanes
    starts_log = [rng.randrange(1, B.n) for _ in range(lanes)]
    cur_pts = mont_pts(B, [E.ec_mul(B, x, B.G) for x in starts_log])
    incs = [mont_pts(B, [seeds[1 + k]] * lanes) for k in range(5)]
    all_x, all_y, all_logs = [], [], []
    cur_logs = list(starts_log)
    for step in range(per):
        cur_pts = ctx.batch_padd(cur_pts, incs[step % 5])
        cur_logs = [(x + d[1 + step % 5]) % B.n for x in cur_logs]
        all_x.append(cur_pts[0]); all_y.append(cur_pts[1]); all_logs += cur_logs
    PX = np.ascontiguousarray(np.concatenate(all_x, axis=1))
    PY = np.ascontiguousarray(np.concatenate(all_y, axis=1))
    PI = np.zeros(n, np.uint8)
    end = from_mont_pts(B, cur_pts)
    assert end[0] == E.ec_mul(B, cur_logs[0], B.G) and end[-1] == E.ec_mul(B, cur_logs[-1], B.G)
    ks = [rng.randrange(1 << 256) for _ in range(n)]
    got = from_mont_pts(B, ctx.msm(cols(ks, 8), (PX, PY, PI)))
    total = sum((k % B.n) * l for k, l in zip(ks, all_logs)) % B.n
    assert got == [E.ec_mul(B, total, B.G)]
