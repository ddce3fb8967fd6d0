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
from tests.util import CURVE_IDS, cols_hex, golden, hex_cols, pts_from_hex, pts_to_hex

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
