"""CPU tests of the product's 12-limb (381 / 377-bit) field layer and the BLS12-381 / BLS12-377
G1 point formulas, compiled for the host (tests/hostsim), against Python integers.

The reference is 256-bit only (limbs.hpp:17), so there is no reference output for this
field: parity is against the definition (north_star's "381-bit Montgomery field")."""
import random

import numpy as np

import paper_2501_03245_b200.capi as G
from oracle import pyec as E
from tests.hostsim import hostsim as H

import pytest

R12 = 1 << 384
BLS = [E.BLS12_381, E.BLS12_377]


def cols(vals, limbs=12):
    return G.cols_from_ints(vals, limbs)


def ints(c):
    return G.ints_from_cols(c)


def edge_values(q, rng, n):
    return [0, 1, 2, q - 1, q - 2, (q + 1) // 2, (1 << 376) % q, (1 << 255) - 19, 0xFFFFFFFF, 1 << 32,
            (1 << 352) - 1] + [rng.randrange(q) for _ in range(n)]


@pytest.mark.parametrize("B", BLS, ids=lambda c: c.name)
def test_field12_ops_vs_python_ints(B):
    q = B.p
    rng = random.Random(381)
    a = edge_values(q, rng, 3000)
    b = list(reversed(edge_values(q, rng, 3000)))
    A, Bc = cols(a), cols(b)
    f = H.BLS_FIELDS[B.cid][0]
    rinv = pow(R12, -1, q)
    assert ints(H.field_op(0, 0, "mont_mul", A, Bc, field_id=f)) == [x * y * rinv % q for x, y in zip(a, b)]
    assert ints(H.field_op(0, 0, "sqr", A, field_id=f)) == [x * x * rinv % q for x in a]
    assert ints(H.field_op(0, 0, "mod_add", A, Bc, field_id=f)) == [(x + y) % q for x, y in zip(a, b)]
    assert ints(H.field_op(0, 0, "mod_sub", A, Bc, field_id=f)) == [(x - y) % q for x, y in zip(a, b)]
    assert ints(H.field_op(0, 0, "to_mont", A, field_id=f)) == [x * R12 % q for x in a]
    assert ints(H.field_op(0, 0, "from_mont", A, field_id=f)) == [x * rinv % q for x in a]
    # inversions: safegcd on plain residues, safegcd and Fermat on Montgomery-form elements
    want_plain = [pow(x, -1, q) if x else 0 for x in a]
    assert ints(H.field_op(0, 0, "inv_plain", A, field_id=f)) == want_plain
    want_mont = [pow(x * rinv % q, -1, q) * R12 % q if x else 0 for x in a]
    assert ints(H.field_op(0, 0, "inv_safegcd", A, field_id=f)) == want_mont
    assert ints(H.field_op(0, 0, "inv_var_plain", A, field_id=f)) == want_plain
    assert ints(H.field_op(0, 0, "inv_sched_plain", A, field_id=f)) == want_plain
    assert ints(H.field_op(0, 0, "inv_sched_exit_plain", A, field_id=f)) == want_plain
    assert ints(H.field_op(0, 0, "inv_var", A, field_id=f)) == want_mont
    small = cols(a[:40])
    assert ints(H.field_op(0, 0, "mod_inv", small, field_id=f)) == want_mont[:40]


@pytest.mark.parametrize("B", BLS, ids=lambda c: c.name)
def test_scalar_field_bls_r(B):
    q = B.n
    rng = random.Random(255)
    a = [0, 1, q - 1, q - 2] + [rng.randrange(q) for _ in range(500)]
    b = list(reversed(a))
    A, Bc = cols(a, 8), cols(b, 8)
    rinv = pow(1 << 256, -1, q)
    f = H.BLS_FIELDS[B.cid][1]
    assert ints(H.field_op(0, 0, "mont_mul", A, Bc, field_id=f)) == [x * y * rinv % q for x, y in zip(a, b)]
    assert ints(H.field_op(0, 0, "inv_plain", A, field_id=f)) == [pow(x, -1, q) if x else 0 for x in a]
    assert ints(H.field_op(0, 0, "inv_var_plain", A, field_id=f)) == [pow(x, -1, q) if x else 0 for x in a]


def mont_pts(B, pts):
    """affine int points (None = infinity) -> Montgomery-form column buffers"""
    xs = [0 if p is None else p[0] * R12 % B.p for p in pts]
    ys = [0 if p is None else p[1] * R12 % B.p for p in pts]
    return cols(xs), cols(ys), np.array([p is None for p in pts], np.uint8)


def from_mont_pts(B, P):
    rinv = pow(R12, -1, B.p)
    xs, ys = ints(P[0]), ints(P[1])
    return [None if P[2][i] else (xs[i] * rinv % B.p, ys[i] * rinv % B.p) for i in range(len(xs))]


@pytest.mark.parametrize("B", BLS, ids=lambda c: c.name)
def test_bls_g1_point_formulas(B):
    rng = random.Random(12381)
    assert E.on_curve(B, B.G)
    base = [E.ec_mul(B, rng.randrange(1, B.n), B.G) for _ in range(24)]
    P = base + [base[0], base[1], None, base[3], None]
    T = list(reversed(base)) + [base[0], (base[1][0], B.p - base[1][1]), base[2], None, None]
    got = from_mont_pts(B, H.bls_point_op("add", mont_pts(B, P), mont_pts(B, T), curve=B.cid))
    assert got == [E.ec_add(B, a, b) for a, b in zip(P, T)]
    got = from_mont_pts(B, H.bls_point_op("dbl", mont_pts(B, P), curve=B.cid))
    assert got == [E.ec_add(B, a, a) for a in P]
    ks = [0, 1, 2, B.n - 1, B.n, (1 << 256) - 1] + [rng.randrange(1 << 256) for _ in range(6)]
    pts = [base[i % len(base)] for i in range(len(ks))]
    got = from_mont_pts(B, H.bls_point_op("mul", mont_pts(B, pts), k=cols(ks, 8), curve=B.cid))
    assert got == [E.ec_mul(B, k, p) for k, p in zip(ks, pts)]
    assert E.ec_mul(B, B.n, B.G) is None  # the generator has order n
