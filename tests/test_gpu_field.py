"""GPU parity of the field layer through the C ABI:
gecc_field_op on the B200 vs the C oracle on the same seeded inputs, plus the
golden vectors generated from the compiled reference."""
import random

import numpy as np
import pytest

import paper_2501_03245_b200 as gecc
from oracle import coracle as O
from tests.util import CURVE_IDS, cols_hex, golden, hex_cols

pytestmark = pytest.mark.gpu
FIELD = golden("field")


@pytest.fixture(scope="module")
def ctxs():
    c = {0: gecc.Context(gecc.SM2), 1: gecc.Context(gecc.SECP256K1)}
    yield c
    for x in c.values():
        x.close()


@pytest.mark.parametrize("key", [k for k in FIELD if not k.startswith("_")])
def test_field_golden_gpu(ctxs, key):
    ent = FIELD[key]
    cid = CURVE_IDS[key.split(".")[0]]
    which = 0 if key.endswith(".p") else 1
    A, B = hex_cols(ent["a"]), hex_cols(ent["b"])
    for op in ("mont_mul", "mod_add", "mod_sub", "to_mont", "from_mont", "mod_inv"):
        assert cols_hex(ctxs[cid].field_op(which, op, A, B)) == ent[op], op


@pytest.mark.parametrize("cid", [0, 1])
@pytest.mark.parametrize("which", [0, 1])
def test_field_random_vs_oracle(ctxs, cid, which):
    """test_field.cpp:63-75 does 50 000 mont_mul per field against its oracle."""
    q = O.field_params(cid, which)["q"]
    rng = random.Random(1000 + 2 * cid + which)
    n = 50_000
    edge = [0, 1, q - 1, q - 2, 2, (1 << 255) % q]
    a = gecc.cols_from_ints(edge + [rng.randrange(q) for _ in range(n - len(edge))])
    b = gecc.cols_from_ints(list(reversed(edge)) + [rng.randrange(q) for _ in range(n - len(edge))])
    for op in ("mont_mul", "mod_add", "mod_sub", "to_mont", "from_mont"):
        got = ctxs[cid].field_op(which, op, a, b)
        want = O.field_op(cid, which, op, a, b)
        bad = np.where((got != want).any(axis=0))[0]
        assert len(bad) == 0, (op, bad[:4])
    m = 512
    a2 = np.ascontiguousarray(a[:, :m])
    assert (ctxs[cid].field_op(which, "mod_inv", a2) == O.field_op(cid, which, "mod_inv", a2)).all()
    # the warp-cooperative inversion (the one shared inversion of the block-level Montgomery trick),
    # ragged count so that the last warp is partly out of range
    a3 = np.ascontiguousarray(a[:, :m + 13])
    assert (ctxs[cid].field_op(which, "mod_inv_warp", a3) == O.field_op(cid, which, "mod_inv", a3)).all()


def test_field_properties_large(ctxs):
    """size-independent properties at 2^20 elements: (a*b)*c == a*(b*c), a*inv-free identities."""
    n = 1 << 20
    rs = np.random.RandomState(7)
    for cid in (0, 1):
        ctx = ctxs[cid]
        a, b, c = (rs.randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32) for _ in range(3))
        for x in (a, b, c):
            x[7] &= 0x7FFFFFFF  # below every modulus used here
        ab_c = ctx.field_op(0, "mont_mul", ctx.field_op(0, "mont_mul", a, b), c)
        a_bc = ctx.field_op(0, "mont_mul", a, ctx.field_op(0, "mont_mul", b, c))
        assert (ab_c == a_bc).all()
        s = ctx.field_op(0, "mod_sub", ctx.field_op(0, "mod_add", a, b), b)
        assert (s == a).all()
        rt = ctx.field_op(0, "from_mont", ctx.field_op(0, "to_mont", a))
        assert (rt == a).all()
