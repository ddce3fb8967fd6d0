"""GPU parity of the batch layer through the C ABI:
batch_invert / batch_padd / batch_pdbl / batch_fpmul / batch_upmul on the B200
against the golden vectors from the compiled reference and the C oracle."""
import random

import numpy as np
import pytest

import paper_2501_03245_b200 as gecc
from oracle import coracle as O
from oracle import pyec as E
from tests.util import CURVE_IDS, cols_hex, golden, hex_cols, pts_from_hex, pts_to_hex

pytestmark = pytest.mark.gpu
BATCH = golden("batch")
CURVES = ["sm2", "secp256k1"]


@pytest.fixture(scope="module")
def ctxs():
    c = {0: gecc.Context(gecc.SM2), 1: gecc.Context(gecc.SECP256K1)}
    yield c
    for x in c.values():
        x.close()


@pytest.fixture(params=["chunked", "coop", "coop32", "tiled8", "tiled4", "fused", "fused2"])
def form(request):
    """Both forms of the batch kernels (one inversion per thread / one per block) must agree
    with the reference bit for bit (results are grouping-invariant, batch_invert.hpp:59-60)."""
    gecc.set_batch_form(request.param)
    yield request.param
    gecc.set_batch_form("auto")


def same(A, B):
    return all((a == b).all() for a, b in zip(A, B))


@pytest.mark.parametrize("name", CURVES)
def test_batch_golden_gpu(ctxs, name, form):
    ent, cid = BATCH[name], CURVE_IDS[name]
    ctx = ctxs[cid]
    P, T = pts_from_hex(ent["P"]), pts_from_hex(ent["T"])
    # exceptional lanes 3/7/11/19/23/31/47 (test_batch_point.cpp:70-100)
    assert pts_to_hex(ctx.batch_padd(P, T)) == ent["padd"]
    assert pts_to_hex(ctx.batch_pdbl(P)) == ent["pdbl"]
    for which in (0, 1):  # zero masking (test_batch_invert.cpp:147-170)
        assert cols_hex(ctx.batch_invert(which, hex_cols(ent[f"inv_in_{which}"]))) == ent[f"inv_out_{which}"]
    assert not ctx.batch_invert(0, np.zeros((8, 5), np.uint32)).any()
    S = hex_cols(ent["edge_scalars"])  # 0, 1, 2^77, n-1, raw all-ones ...
    assert pts_to_hex(ctx.batch_fpmul(S)) == ent["fpmul_edge"]
    assert pts_to_hex(ctx.batch_upmul(S, pts_from_hex(ent["upmul_Q"]))) == ent["upmul_edge"]


@pytest.mark.parametrize("cid", [0, 1])
def test_batch_random_vs_oracle(ctxs, cid, form):
    c, ctx = E.CURVES[cid], ctxs[cid]
    rng = random.Random(300 + cid)
    n = 1500
    k1 = gecc.cols_from_ints([rng.randrange(1 << 256) for _ in range(n)])
    k2 = gecc.cols_from_ints([rng.randrange(1, c.n) for _ in range(n)])
    P = ctx.batch_fpmul(k1)
    assert same(P, O.batch_fpmul(cid, k1, lanes=16))
    T = ctx.batch_fpmul(k2)
    assert same(ctx.batch_padd(P, T), O.batch_padd(cid, P, T, lanes=7))
    assert same(ctx.batch_pdbl(P), O.batch_pdbl(cid, P, lanes=7))
    m = 300
    Ps = tuple(np.ascontiguousarray(a[..., :m]) for a in P)
    ks = np.ascontiguousarray(k2[:, :m])
    assert same(ctx.batch_upmul(ks, Ps), O.pmul_serial(cid, ks, Ps))
    for which, q in ((0, c.p), (1, c.n)):
        a = gecc.cols_from_ints([0 if i % 41 == 0 else rng.randrange(1, q) for i in range(5000)])
        assert (ctx.batch_invert(which, a) == O.batch_invert(cid, which, a, lanes=9)).all()


def test_batch_sizes_and_errors(ctxs, form):
    ctx = ctxs[1]
    empty = (np.zeros((8, 0), np.uint32), np.zeros((8, 0), np.uint32), np.zeros(0, np.uint8))
    assert ctx.batch_padd(empty, empty)[0].shape == (8, 0)  # empty batches are fine
    assert ctx.batch_invert(0, np.zeros((8, 0), np.uint32)).shape == (8, 0)
    one = (np.zeros((8, 1), np.uint32), np.zeros((8, 1), np.uint32), np.zeros(1, np.uint8))
    with pytest.raises(ValueError):  # batch_point.cpp:71-72
        ctx.batch_padd(one, empty)
    # ragged sizes around the chunking boundaries: all-infinity + t = infinity returns p
    rng = random.Random(4)
    for n in (1, 2, 127, 128, 129, 1023, 1024, 1025, 2049):
        k = gecc.cols_from_ints([rng.randrange(1, E.SECP256K1.n) for _ in range(n)])
        P = ctx.batch_fpmul(k)
        inf = (np.zeros((8, n), np.uint32), np.zeros((8, n), np.uint32), np.ones(n, np.uint8))
        assert same(ctx.batch_padd(P, inf), P)      # test_batch_point.cpp:102-112
        assert same(ctx.batch_padd(inf, P), P)
        assert ctx.batch_padd(inf, inf)[2].all()
        negP = (P[0], gecc.cols_from_ints([(E.SECP256K1.p - y) % E.SECP256K1.p for y in gecc.ints_from_cols(P[1])]), P[2])
        assert ctx.batch_padd(P, negP)[2].all()     # p + (-p) = infinity
        assert same(ctx.batch_padd(P, P), ctx.batch_pdbl(P))


def test_padd_properties_large(ctxs, form):
    """2^20 pairs: commutativity and (P+T)+(-T) == P, plus a CPU spot check."""
    ctx, c = ctxs[1], E.SECP256K1
    n = 1 << 20
    rs = np.random.RandomState(11)
    k1 = rs.randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32)
    k2 = rs.randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32)
    P, T = ctx.batch_fpmul(k1), ctx.batch_fpmul(k2)
    S = ctx.batch_padd(P, T)
    assert same(S, ctx.batch_padd(T, P))
    negT = ctx.field_op(0, "mod_sub", np.zeros((8, n), np.uint32), T[1])
    back = ctx.batch_padd(S, (T[0], negT, T[2]))
    assert same(back, P)
    idx = rs.choice(n, 64, replace=False)
    sub = lambda A: tuple(np.ascontiguousarray(a[..., idx]) for a in A)
    assert same(sub(S), O.batch_padd(1, sub(P), sub(T)))
