"""GPU parity tests added in round 2 (VERDICT r01 "close the non-inherent parity gaps" and the
second boundary): config 1 at its stated size, the reduce-edge vectors and the weakly reduced
secp256k1 field ON the GPU, group contexts (one context, several device shards), explicit-nonce
signing, arbitrary-base tables, the constant-structure mode and the NCCL exchange of the
sharded MSM with a one-rank communicator.  Everything goes through the C ABI."""
import ctypes as C
import random

import numpy as np
import pytest

import paper_2501_03245_b200 as gecc
from oracle import coracle as O
from oracle import pyec as E
from tests.util import CURVE_IDS, cols_hex, golden, hex_cols, pts_from_hex, pts_to_hex, wide_cols

pytestmark = pytest.mark.gpu
FIELD, BATCH, ECDSA = golden("field"), golden("batch"), golden("ecdsa")
CURVES = ["sm2", "secp256k1"]


@pytest.fixture(scope="module")
def ctxs():
    c = {0: gecc.Context(gecc.SM2), 1: gecc.Context(gecc.SECP256K1)}
    yield c
    for x in c.values():
        x.close()


@pytest.fixture(scope="module")
def groups():
    """Group contexts with three shards on device 0: the sharding logic of a multi-GPU box,
    exercised on the one GPU this box has."""
    c = {0: gecc.Context(gecc.SM2, devices=[0, 0, 0]), 1: gecc.Context(gecc.SECP256K1, devices=[0, 0, 0])}
    yield c
    for x in c.values():
        x.close()


def same(A, B):
    return all((a == b).all() for a, b in zip(A, B))


# ------------------------------------------------------------------ config 1 at its stated size
@pytest.mark.parametrize("form", ["auto", "chunked", "tiled8", "fused"])
def test_config1_padd_2p16_vs_oracle(ctxs, form):
    """BASELINE config 1: secp256k1 batched affine addition, 2^16 random pairs, EVERY lane
    compared with the CPU oracle, with the exceptional-lane fixture (P = T, P = -T, infinity
    operands; test_batch_point.cpp:70-100) spliced in at the start, across a tile boundary and
    at the end."""
    ent = BATCH["secp256k1"]
    n = 1 << 16
    rng = np.random.RandomState(2016)
    k = rng.randint(0, 2**32, size=(8, 2 * n), dtype=np.uint64).astype(np.uint32)
    ctx = ctxs[1]
    pts = ctx.batch_fpmul(np.ascontiguousarray(k))
    P = [np.ascontiguousarray(a[..., :n]) for a in pts]
    T = [np.ascontiguousarray(a[..., n:]) for a in pts]
    fp, ft = pts_from_hex(ent["P"]), pts_from_hex(ent["T"])
    m = fp[0].shape[1]
    for at in (0, 2048 - 20, n - m):
        for dst, src in ((P, fp), (T, ft)):
            dst[0][:, at:at + m] = src[0]
            dst[1][:, at:at + m] = src[1]
            dst[2][at:at + m] = src[2]
    gecc.set_batch_form(form)
    try:
        got = ctx.batch_padd(tuple(P), tuple(T))
    finally:
        gecc.set_batch_form("auto")
    want = O.batch_padd(1, tuple(P), tuple(T), lanes=64, workers=8)
    assert same(got, want)
    assert pts_to_hex(tuple(np.ascontiguousarray(a[..., :m]) for a in got)) == ent["padd"]
    assert got[2].sum() >= 3     # the fixture's infinity results are present in every splice


# ------------------------------------------------------------------ reduce edges, lazy field
@pytest.mark.parametrize("key", [k for k in FIELD if not k.startswith("_")])
def test_mont_reduce_edges_gpu(ctxs, key):
    """512-bit reduce-edge vectors (test_field.cpp:136-164) through mont_reduce ON the GPU: the
    secp256k1 word-serial route, the SM2 add/sub-only route and the generic word-serial route."""
    ent = FIELD[key]
    cid = CURVE_IDS[key.split(".")[0]]
    which = 0 if key.endswith(".p") else 1
    q = int(ent["q"], 16)
    rng = random.Random(78)
    extra = [format(rng.randrange(q << 256), "0128x") for _ in range(20000)]
    c16 = wide_cols(ent["reduce_in"] + extra)
    lo, hi = np.ascontiguousarray(c16[:8]), np.ascontiguousarray(c16[8:])
    got = ctxs[cid].field_op(which, "mont_reduce", lo, hi)
    assert cols_hex(got)[:len(ent["reduce_in"])] == ent["reduce_generic"]
    assert (got == O.mont_reduce(cid, which, c16, False)).all()


def test_lazy_secp_field_gpu(ctxs):
    """The weakly reduced plain secp256k1 field the headline kernel computes in, directly:
    non-canonical inputs (q, q + 1, 2^256 - 1 ...) and every pair of the edge values that drive
    the rare carry / borrow branches of the folds, against Python integers."""
    p = E.SECP256K1.p
    rng = random.Random(12)
    special = [0, 1, p - 1, p, p + 1, 2**256 - 1, 2**256 - 2, p + 977, 2**255, 2**256 - 2**32, 2**256 - 977, 5]
    edge = special + [2**64 - 1, 2**64, 2**64 - 977, 2**256 - 2**64, 2**256 - 2**64 + 1, 977, 976, 2**32 + 977,
                      2**32 + 976, 2**256 - 2**32 - 978, (1 << 256) - (1 << 33), 2**96 - 1]
    a = [x for x in edge for _ in edge] + [rng.randrange(1 << 256) for _ in range(50000)]
    b = [y for _ in edge for y in edge] + [rng.randrange(1 << 256) for _ in range(50000)]
    A, B = gecc.cols_from_ints(a), gecc.cols_from_ints(b)
    ctx = ctxs[1]
    for op, fn in (("lazy_mul", lambda x, y: x * y), ("lazy_sqr", lambda x, y: x * x),
                   ("lazy_add", lambda x, y: x + y), ("lazy_sub", lambda x, y: x - y)):
        got = gecc.ints_from_cols(ctx.field_op(0, op, A, B))
        bad = [i for i, (g, x, y) in enumerate(zip(got, a, b)) if g != fn(x, y) % p]
        assert not bad, (op, bad[:4])
    with pytest.raises(ValueError):     # the representation exists for the secp256k1 base field only
        ctx.field_op(1, "lazy_mul", A, B)
    with pytest.raises(ValueError):
        ctxs[0].field_op(0, "lazy_mul", A, B)


# ------------------------------------------------------------------ group contexts
@pytest.mark.parametrize("name", CURVES)
def test_group_context_equals_device_context(ctxs, groups, name):
    """One context driving several device shards returns the bytes of a one-device call: lanes
    are split into contiguous ranges, the nonce stream id stays the global lane index."""
    ent, cid = ECDSA[name], CURVE_IDS[name]
    ctx, grp = ctxs[cid], groups[cid]
    assert grp.shards == 3 and ctx.shards == 1
    n = 1000      # not a multiple of 3: ragged ranges
    rc, sec, pub = grp.keygen(5, n)
    assert (rc, sec, pub) == ctx.keygen(5, n)
    dig = np.random.RandomState(4).bytes(32 * n)
    assert grp.sign(dig, sec, 7) == ctx.sign(dig, sec, 7)
    assert grp.sign(dig, sec, 7, lane_base=12345) == ctx.sign(dig, sec, 7, lane_base=12345)
    sig = bytearray(ctx.sign(dig, sec, 7)[1])
    for i in (0, 333, 334, 999):
        sig[64 * i + 5] ^= 1
    want = ctx.verify(dig, pub, bytes(sig))
    assert grp.verify(dig, pub, bytes(sig)) == want and sum(want[1]) == n - 4
    peers = pub[65:] + pub[:65]
    assert grp.ecdh(sec, peers) == ctx.ecdh(sec, peers)
    # golden records through the group
    gsec, gpub = bytes.fromhex(ent["secrets"]), bytes.fromhex(ent["publics"])
    gdig, gsig = bytes.fromhex(ent["digests"]), bytes.fromhex(ent["sigs"])
    assert grp.keygen(ent["keygen_seed"], ent["n"]) == (0, gsec, gpub)
    assert grp.sign(gdig, gsec, ent["nonce_seed"]) == (0, gsig, [0] * ent["n"])
    # ledger: the closed forms of ONE call over the whole batch, not a sum of shards
    grp.ledger_reset(); ctx.ledger_reset()
    grp.sign(dig, sec, 7); ctx.sign(dig, sec, 7)
    assert grp.ledger() == ctx.ledger() and grp.ledger()["modinv"] == 257
    # a zero secret anywhere fails the whole call (capi.cpp:181-184), whichever shard sees it
    bad_sec = bytearray(sec)
    bad_sec[32 * 700:32 * 701] = bytes(32)
    assert grp.sign(dig, bytes(bad_sec), 7)[0] == 2
    # first failing lane's code when no lane_status is passed (capi.cpp:64-73)
    bad_peers = bytearray(peers)
    bad_peers[65 * 800 + 40] ^= 1
    assert grp.ecdh(sec, bytes(bad_peers), want_status=False)[0] == ctx.ecdh(sec, bytes(bad_peers), want_status=False)[0] == 3


@pytest.mark.parametrize("cid", [0, 1])
def test_group_context_batch_layer(ctxs, groups, cid):
    ctx, grp = ctxs[cid], groups[cid]
    rng = np.random.RandomState(70 + cid)
    n = 4099
    k = rng.randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32)
    k2 = rng.randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32)
    P = ctx.batch_fpmul(k)
    assert same(grp.batch_fpmul(k), P)
    T = ctx.batch_fpmul(k2)
    T[2][5] = 1; T[0][:, 5] = 0; T[1][:, 5] = 0            # an infinity operand
    T[0][:, 2000] = P[0][:, 2000]; T[1][:, 2000] = P[1][:, 2000]   # P == T: tangent lane
    assert same(grp.batch_padd(P, T), ctx.batch_padd(P, T))
    assert same(grp.batch_pdbl(P), ctx.batch_pdbl(P))
    m = 300
    cut = lambda A: tuple(np.ascontiguousarray(a[..., :m]) for a in A)
    assert same(grp.batch_upmul(np.ascontiguousarray(k2[:, :m]), cut(P)), ctx.batch_upmul(np.ascontiguousarray(k2[:, :m]), cut(P)))
    for which in (0, 1):
        q = O.field_params(cid, which)["q"]
        a = gecc.cols_from_ints([0, 1, q - 1] + [random.Random(3).randrange(q) for _ in range(500)])
        assert (grp.batch_invert(which, a) == ctx.batch_invert(which, a)).all()
        assert (grp.field_op(which, "mont_mul", a, a) == ctx.field_op(which, "mont_mul", a, a)).all()
    # MSM: point ranges per shard, partial sums exchanged and added on the first device
    got = grp.msm(k2, P)
    assert same(got, ctx.msm(k2, P))
    small = 37
    ks = np.ascontiguousarray(k2[:, :small])
    Ps = tuple(np.ascontiguousarray(a[..., :small]) for a in P)
    assert same(grp.msm(ks, Ps), O.msm(cid, ks, Ps))
    # fewer points than shards: empty ranges contribute the point at infinity
    one = (np.ascontiguousarray(P[0][:, :1]), np.ascontiguousarray(P[1][:, :1]), np.zeros(1, np.uint8))
    assert same(grp.msm(np.ascontiguousarray(k2[:, :1]), one), ctx.msm(np.ascontiguousarray(k2[:, :1]), one))


def test_group_dev_entry_points_are_rejected(groups):
    """Device-pointer entry points address one device: invalid on a group context."""
    l, g = gecc.lib(), groups[1]
    assert l.gecc_verify_dev(g.h, C.c_size_t(0), None, None, None, None) == 1
    assert l.gecc_ctx_set_stream(g.h, None) == 1
    assert l.gecc_batch_padd_dev(g.h, C.c_size_t(0), None, None, None, None, None, None, None, None, None) == 1


# ------------------------------------------------------------------ explicit nonces
@pytest.mark.parametrize("name", CURVES)
def test_sign_nonces_gpu(ctxs, groups, name):
    """gecc_sign_nonces (one attempt with caller-supplied nonces) reproduces sm2b_sign when fed
    the deterministic source's attempt-0 nonces; out-of-range nonces and a rigged s == 0 come
    back as 'replace this nonce' (protocol.cpp:121-164)."""
    cid = CURVE_IDS[name]
    c = E.CURVES[cid]
    rng = random.Random(6 + cid)
    n, seed = 257, 21
    sec = b"".join(E.be32(rng.randrange(1, c.n)) for _ in range(n))
    dig = bytearray(rng.randrange(256) for _ in range(32 * n))
    nonces = bytearray(b"".join(E.be32(O.nonce(cid, seed, i, 0)) for i in range(n)))
    want = ctxs[cid].sign(bytes(dig), sec, seed)
    for ctx in (ctxs[cid], groups[cid]):
        assert ctx.sign_nonces(bytes(dig), sec, bytes(nonces)) == want
    nonces[32 * 3:32 * 4] = bytes(32)
    nonces[32 * 4:32 * 5] = E.be32(c.n)
    d6 = int.from_bytes(sec[32 * 6:32 * 7], "big")
    r6 = E.ec_mul(c, O.nonce(cid, seed, 6, 0), c.G)[0] % c.n
    dig[32 * 6:32 * 7] = E.be32((-r6 * d6) % c.n)
    for ctx in (ctxs[cid], groups[cid]):
        rc, sig, st = ctx.sign_nonces(bytes(dig), sec, bytes(nonces))
        assert rc == 0 and [i for i, s in enumerate(st) if s] == [3, 4, 6] and {st[3], st[4], st[6]} == {5}
        for i in (3, 4, 6):
            assert sig[64 * i:64 * i + 64] == bytes(64)
        assert sig[64 * 7:] == want[1][64 * 7:]
        assert ctx.sign_nonces(bytes(dig), sec, bytes(nonces), want_status=False)[0] == 5
        bad = bytearray(sec)
        bad[32 * 200:32 * 201] = E.be32(c.n)      # secret >= n: whole call malformed
        assert ctx.sign_nonces(bytes(dig), bytes(bad), bytes(nonces))[0] == 2


# ------------------------------------------------------------------ base tables
@pytest.mark.parametrize("name", CURVES)
def test_precompute_base_table_arbitrary_base(ctxs, groups, name):
    """precompute_base_table(c, g) for g != G and batch_fpmul over it (batch_point.hpp:76-91,
    test_batch_point.cpp:174-208): scalars[i] * g against the oracle's serial multiplication,
    edge scalars {0, 1, 2^77, n-1, all-ones} included; an off-curve base is rejected."""
    ent, cid = BATCH[name], CURVE_IDS[name]
    c = E.CURVES[cid]
    base_k = gecc.cols_from_ints([0xC0FFEE123456789])
    rng = random.Random(40 + cid)
    S = np.ascontiguousarray(np.concatenate([hex_cols(ent["edge_scalars"]),
                                             gecc.cols_from_ints([rng.randrange(1 << 256) for _ in range(200)])], axis=1))
    n = S.shape[1]
    for ctx in (ctxs[cid], groups[cid]):
        g = ctx.batch_fpmul(base_k)
        tab = ctx.base_table(g[0][:, 0], g[1][:, 0])
        got = ctx.batch_fpmul(S, tab)
        rep = tuple(np.ascontiguousarray(np.repeat(a.reshape(a.shape[0], 1) if a.ndim == 2 else a, n, axis=-1)) for a in g)
        want = O.pmul_serial(cid, S, rep)
        assert same(got, want)
        # the generator's own table gives batch_fpmul's answer
        G = ctx.batch_fpmul(gecc.cols_from_ints([1]))
        gtab = ctx.base_table(G[0][:, 0], G[1][:, 0])
        assert same(ctx.batch_fpmul(S, gtab), ctx.batch_fpmul(S))
        off = g[1][:, 0].copy()
        off[0] ^= 1
        with pytest.raises(ValueError, match="off curve"):
            ctx.base_table(g[0][:, 0], off)
        tab.close(); gtab.close()


# ------------------------------------------------------------------ constant-structure mode
@pytest.mark.parametrize("name", CURVES)
def test_secret_uniform_mode_gpu(name):
    """GECC_SECRET_UNIFORM: k*G (keygen, sign) and d*P (ECDH) with every window's addition
    executed and entries chosen by select -- outputs identical to the fast path and the golden."""
    ent, cid = ECDSA[name], CURVE_IDS[name]
    n = ent["n"]
    sec, pub = bytes.fromhex(ent["secrets"]), bytes.fromhex(ent["publics"])
    dig, sig = bytes.fromhex(ent["digests"]), bytes.fromhex(ent["sigs"])
    with gecc.Context(cid) as ctx:
        m = 3000
        fast = (ctx.keygen(9, m), )
        rdig = np.random.RandomState(8).bytes(32 * m)
        fast += (ctx.sign(rdig, fast[0][1], 11), ctx.ecdh(fast[0][1], fast[0][2][65:] + fast[0][2][:65]))
        ctx.set_secret_mode(gecc.SECRET_UNIFORM)
        assert ctx.keygen(ent["keygen_seed"], n) == (0, sec, pub)
        assert ctx.sign(dig, sec, ent["nonce_seed"]) == (0, sig, [0] * n)
        rt = ent["retry"]
        assert ctx.sign(bytes.fromhex(rt["digests"]), bytes.fromhex(rt["secrets"]), rt["nonce_seed"])[1].hex() == rt["sigs"]
        e = ent["ecdh"]
        got = ctx.ecdh(bytes.fromhex(e["secrets"]), bytes.fromhex(e["peers"]))
        assert (got[1].hex(), got[2]) == (e["shared"], e["status"])
        uni = (ctx.keygen(9, m), )
        uni += (ctx.sign(rdig, uni[0][1], 11), ctx.ecdh(uni[0][1], uni[0][2][65:] + uni[0][2][:65]))
        assert uni == fast
        # edge secrets: 1, 2, n - 1, 2^16, 2^255 (zero digits everywhere but one window)
        c = E.CURVES[cid]
        es = b"".join(E.be32(v) for v in (1, 2, c.n - 1, 1 << 16, 1 << 255 if (1 << 255) < c.n else 1 << 254, (1 << 128) + 1))
        k = len(es) // 32
        ed = np.random.RandomState(9).bytes(32 * k)
        peers = uni[0][2][:65 * k]
        u = (ctx.sign(ed, es, 3), ctx.ecdh(es, peers))
        ctx.set_secret_mode(gecc.SECRET_FAST)
        assert u == (ctx.sign(ed, es, 3), ctx.ecdh(es, peers))
        assert u[0] == O.ecdsa_sign(cid, ed, es, 3)


# ------------------------------------------------------------------ NCCL exchange, one rank
@pytest.mark.parametrize("curve", [gecc.SECP256K1, gecc.BLS12_377])
def test_msm_exchange_over_nccl_one_rank(curve):
    """The multi-process MSM exchange (ncclAllGather of the partial sums + local additions),
    executed for real with a one-rank communicator: the only way to run NCCL on a one-GPU box.
    The combined point must equal the partial sum it started from, infinity included."""
    import torch
    L = 12 if curve == gecc.BLS12_377 else 8
    with gecc.Context(curve, 0) as ctx:
        ctx.comm_init_rank(1, 0, gecc.comm_unique_id())
        l = gecc.lib()
        if curve == gecc.SECP256K1:
            k = gecc.cols_from_ints([5, 7, 11])
            P = ctx.batch_fpmul(k)
            want = ctx.msm(k, P)
        else:
            B = E.CURVES["bls12_377"]
            R = 1 << 384
            want = (gecc.cols_from_ints([B.gx * R % B.p], 12), gecc.cols_from_ints([B.gy * R % B.p], 12), np.zeros(1, np.uint8))
        x = torch.from_numpy(want[0].view(np.int32).copy()).cuda()
        y = torch.from_numpy(want[1].view(np.int32).copy()).cuda()
        inf = torch.from_numpy(want[2].copy()).cuda()
        vp = lambda t: C.c_void_p(t.data_ptr())
        assert l.gecc_msm_combine_dev(ctx.h, vp(x), vp(y), vp(inf)) == 0, l.gecc_last_error(ctx.h)
        torch.cuda.synchronize()
        assert (x.cpu().numpy().view(np.uint32).reshape(L, 1) == want[0]).all()
        assert (y.cpu().numpy().view(np.uint32).reshape(L, 1) == want[1]).all()
        assert int(inf.item()) == 0
        inf.fill_(1)
        assert l.gecc_msm_combine_dev(ctx.h, vp(x), vp(y), vp(inf)) == 0
        torch.cuda.synchronize()
        assert int(inf.item()) == 1 and int(x.abs().sum()) == 0


def test_combine_without_communicator_fails_loudly():
    import torch
    with gecc.Context(gecc.SECP256K1, 0) as ctx:
        z = torch.zeros(8, dtype=torch.int32, device="cuda")
        i = torch.zeros(1, dtype=torch.uint8, device="cuda")
        vp = lambda t: C.c_void_p(t.data_ptr())
        assert gecc.lib().gecc_msm_combine_dev(ctx.h, vp(z), vp(z), vp(i)) == 7
        assert b"communicator" in gecc.lib().gecc_last_error(ctx.h)
