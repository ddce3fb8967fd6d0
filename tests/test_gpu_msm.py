"""GPU MSM.  The reference has no MSM, so parity is
against the definition: the oracle's sum of pmul_serial results at small n, and the
identity sum_i s_i (t_i G) = (sum_i s_i t_i mod n) G at 2^20 (Python ints + fixed-base)."""
import random

import numpy as np
import pytest

import paper_2501_03245_b200 as gecc
from oracle import coracle as O
from oracle import pyec as E

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctxs():
    c = {0: gecc.Context(gecc.SM2), 1: gecc.Context(gecc.SECP256K1)}
    yield c
    for x in c.values():
        x.close()


@pytest.fixture(params=["affine", "affine1", "fused16", "fused8", "jacobian"], autouse=True)
def msm_form(request):
    """every test runs with both bucket-accumulation forms (results must be identical)"""
    gecc.set_msm_form(request.param)
    yield request.param
    gecc.set_msm_form("auto")


def same(A, B):
    return all((np.asarray(a) == np.asarray(b)).all() for a, b in zip(A, B))


@pytest.mark.parametrize("cid", [0, 1])
def test_msm_small_vs_oracle(ctxs, cid):
    ctx, c = ctxs[cid], E.CURVES[cid]
    rng = random.Random(40 + cid)
    for n in (1, 2, 17, 200):
        s = gecc.cols_from_ints([rng.randrange(1 << 256) for _ in range(n)])
        P = ctx.batch_fpmul(gecc.cols_from_ints([rng.randrange(1, c.n) for _ in range(n)]))
        assert same(ctx.msm(s, P), O.msm(cid, s, P)), n
    # edge cases: zero scalars, infinity inputs, the same point many times (bucket collisions
    # force the doubling branch), scalars n-1 / n / 2^256-1, cancelling pairs
    n = 64
    P = list(ctx.batch_fpmul(gecc.cols_from_ints([rng.randrange(1, c.n) for _ in range(n)])))
    for i in range(8, 24):
        for a in (0, 1):
            P[a][:, i] = P[a][:, 8]
    ks = [rng.randrange(c.n) for _ in range(n)]
    ks[0], ks[1], ks[2], ks[3], ks[4] = 0, c.n - 1, c.n, (1 << 256) - 1, 1
    for i in range(8, 24):
        ks[i] = 5
    ks[30], ks[31] = 77, c.n - 77
    ks[5], ks[6], ks[7] = (0x7FFF << 240) | (0x9000 << 224), (1 << 255) - 1, 1 << 255  # recoding-carry window
    for a in (0, 1):
        P[a][:, 31] = P[a][:, 30]
    P[2][40] = 1
    P[0][:, 40] = 0
    P[1][:, 40] = 0
    s = gecc.cols_from_ints(ks)
    assert same(ctx.msm(s, tuple(P)), O.msm(cid, s, tuple(P)))
    # everything cancels -> infinity; empty sum -> infinity
    z = gecc.cols_from_ints([0] * 5)
    five = tuple(np.ascontiguousarray(a[..., :5]) for a in P)
    assert ctx.msm(z, five)[2][0] == 1
    empty = (np.zeros((8, 0), np.uint32), np.zeros((8, 0), np.uint32), np.zeros(0, np.uint8))
    assert ctx.msm(np.zeros((8, 0), np.uint32), empty)[2][0] == 1


def test_msm_identity_2_20(ctxs):
    ctx, c = ctxs[1], E.SECP256K1
    n = 1 << 20
    rs = np.random.RandomState(21)
    t = rs.randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32)
    s = rs.randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32)
    P = ctx.batch_fpmul(t)
    got = ctx.msm(s, P)
    ti = [v % c.n for v in gecc.ints_from_cols(t)]
    si = [v % c.n for v in gecc.ints_from_cols(s)]
    total = sum(a * b for a, b in zip(si, ti)) % c.n
    want = ctx.batch_fpmul(gecc.cols_from_ints([total]))
    assert same(got, want)
    # linearity: MSM over the two halves adds up to the whole
    h = n // 2
    cut = lambda a, lo, hi: np.ascontiguousarray(a[..., lo:hi])
    a = ctx.msm(cut(s, 0, h), tuple(cut(x, 0, h) for x in P))
    b = ctx.msm(cut(s, h, n), tuple(cut(x, h, n) for x in P))
    assert same(ctx.batch_padd(a, b), got)


@pytest.mark.parametrize("cid", [0, 1])
def test_msm_skewed_buckets(ctxs, cid):
    """Runs far longer than a tree node: one scalar for every point (17 runs of n entries),
    a handful of distinct scalars, the same point everywhere (tangent joins at every level),
    and alternating P / -P (every join cancels)."""
    ctx, c = ctxs[cid], E.CURVES[cid]
    rng = random.Random(50 + cid)
    n = 1500
    P = ctx.batch_fpmul(gecc.cols_from_ints([rng.randrange(1, c.n) for _ in range(n)]))
    k = rng.randrange(1, c.n)
    for ks in ([k] * n, [rng.choice([k, 3, c.n - 3, 1 << 200]) for _ in range(n)]):
        s = gecc.cols_from_ints(ks)
        assert same(ctx.msm(s, P), O.msm(cid, s, P))
    Q = tuple(np.ascontiguousarray(np.repeat(a[..., :1], n, axis=-1)) for a in P)
    s = gecc.cols_from_ints([k] * n)
    assert same(ctx.msm(s, Q), O.msm(cid, s, Q))
    s = gecc.cols_from_ints([k if i % 2 == 0 else c.n - k for i in range(n)])
    assert ctx.msm(s, Q)[2][0] == 1
    s = gecc.cols_from_ints([k if i % 2 == 0 else c.n - k for i in range(n - 1)] + [0])
    got = ctx.msm(s, Q)
    one = tuple(np.ascontiguousarray(a[..., :1]) for a in Q)
    assert same(got, O.msm(cid, gecc.cols_from_ints([k]), one))
