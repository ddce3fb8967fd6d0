"""TEST INFRASTRUCTURE ONLY -- textbook affine EC arithmetic and ECDSA on Python ints.

Independent of every other implementation in this repository (shares no limb
code with oracle/gecc_oracle.c, the CUDA kernels or the reference).  It restates
the reference's *test* oracle, /root/reference/proj/tests/ec_oracle.hpp:31-80
(ec_add / ec_mul / ecdsa_sign / ecdsa_verify over boost cpp_int), and its
deterministic nonce recipe, proj/src/protocol.cpp:13-34,67-75, for both curves.

Only tests/, __graft_entry__.smoke() and bench.py's CPU arm may import this.
"""
from __future__ import annotations

from dataclasses import dataclass

MASK64 = (1 << 64) - 1


@dataclass(frozen=True)
class Curve:
    name: str
    cid: int
    p: int
    a: int
    b: int
    n: int
    gx: int
    gy: int

    @property
    def G(self):
        return (self.gx, self.gy)


# ec_oracle.hpp:15-24 (SM2 constants as hex strings) / curve.cpp:11-18, field.cpp:10-15
SM2 = Curve(
    "sm2", 0,
    p=2**256 - 2**224 - 2**96 + 2**64 - 1,
    a=2**256 - 2**224 - 2**96 + 2**64 - 1 - 3,
    b=0x28E9FA9E9D9F5E344D5A9E4BCF6509A7F39789F515AB8F92DDBCBD414D940E93,
    n=0xFFFFFFFEFFFFFFFFFFFFFFFFFFFFFFFF7203DF6B21C6052B53BBF40939D54123,
    gx=0x32C4AE2C1F1981195F9904466A39C9948FE30BBFF2660BE1715A4589334C74C7,
    gy=0xBC3736A2F4F6779C59BDCEE36B692153D0A9877CC62A474002DF32E52139F0A0,
)

# SEC 2 v2, section 2.4.1 (SURVEY.md section 8c lists the same constants)
SECP256K1 = Curve(
    "secp256k1", 1,
    p=2**256 - 2**32 - 977,
    a=0,
    b=7,
    n=0xFFFFFFFFFFFFFFFFFFFFFFFFFFFFFFFEBAAEDCE6AF48A03BBFD25E8CD0364141,
    gx=0x79BE667EF9DCBBAC55A06295CE870B07029BFCDB2DCE28D959F2815B16F81798,
    gy=0x483ADA7726A3C4655DA4FBFC0E1108A8FD17B448A68554199C47D08FFB10D4B8,
)

# BLS12-381 G1 (the pairing-friendly curve of north_star's 381-bit field; not in the reference,
# which is 256-bit only): y^2 = x^3 + 4 over the 381-bit prime, prime-order subgroup of order n,
# standard generator (draft-irtf-cfrg-pairing-friendly-curves, section 4.2.1).
BLS12_381 = Curve(
    "bls12_381", 2,
    p=0x1a0111ea397fe69a4b1ba7b6434bacd764774b84f38512bf6730d2a0f6b0f6241eabfffeb153ffffb9feffffffffaaab,
    a=0,
    b=4,
    n=0x73eda753299d7d483339d80809a1d80553bda402fffe5bfeffffffff00000001,
    gx=0x17f1d3a73197d7942695638c4fa9ac0fc3688c4f9774b905a14e3a3f171bac586c55e83ff97a1aeffb3af00adb22c6bb,
    gy=0x08b3f481e3aaa0f1a09e30ed741d8ae4fcf5e095d5d00af600db18cb2c04b3edd03cc744a2888ae40caa232946c5e7e1,
)

# BLS12-377 G1 (BASELINE.json config 4 names it): y^2 = x^3 + 1 over the 377-bit prime, group order
# the 253-bit n, the arkworks / Zexe generator.
BLS12_377 = Curve(
    "bls12_377", 3,
    p=0x01ae3a4617c510eac63b05c06ca1493b1a22d9f300f5138f1ef3622fba094800170b5d44300000008508c00000000001,
    a=0,
    b=1,
    n=0x12ab655e9a2ca55660b44d1e5c37b00159aa76fed00000010a11800000000001,
    gx=0x008848defe740a67c8fc6225bf87ff5485951e2caa9d41bb188282c8bd37cb5cd5481512ffcd394eeab9b16eb21be9ef,
    gy=0x01914a69c5102eff1f674f5d30afeec4bd7fb348ca3e52d96d182ad44fb82305c2fe3d3634a9591afd82de55559c8ea6,
)

CURVES = {0: SM2, 1: SECP256K1, 2: BLS12_381, 3: BLS12_377, "sm2": SM2, "secp256k1": SECP256K1,
          "bls12_381": BLS12_381, "bls12_377": BLS12_377}

INF = None  # point at infinity


def on_curve(c: Curve, pt) -> bool:
    if pt is INF:
        return True
    x, y = pt
    return (y * y - (x * x * x + c.a * x + c.b)) % c.p == 0


def ec_add(c: Curve, A, B):
    """ec_oracle.hpp:31-48 -- complete affine addition."""
    if A is INF:
        return B
    if B is INF:
        return A
    if A[0] == B[0]:
        if (A[1] + B[1]) % c.p == 0:
            return INF
        lam = (3 * A[0] * A[0] + c.a) * pow(2 * A[1], -1, c.p) % c.p
    else:
        lam = (A[1] - B[1]) * pow(A[0] - B[0], -1, c.p) % c.p
    xr = (lam * lam - A[0] - B[0]) % c.p
    yr = (lam * (A[0] - xr) - A[1]) % c.p
    return (xr, yr)


def ec_neg(c: Curve, A):
    return INF if A is INF else (A[0], (-A[1]) % c.p)


def ec_mul(c: Curve, k: int, P):
    """ec_oracle.hpp:50-58 -- LSB-first double-and-add (k taken as given, not reduced)."""
    acc = INF
    while k > 0:
        if k & 1:
            acc = ec_add(c, acc, P)
        P = ec_add(c, P, P)
        k >>= 1
    return acc


def ecdsa_sign(c: Curve, e: int, d: int, k: int):
    """ec_oracle.hpp:62-68"""
    R = ec_mul(c, k, c.G)
    r = R[0] % c.n
    s = pow(k, -1, c.n) * ((e + r * d) % c.n) % c.n
    return r, s


def ecdsa_verify(c: Curve, e: int, pub, r: int, s: int) -> bool:
    """ec_oracle.hpp:70-80"""
    if not (0 < r < c.n and 0 < s < c.n) or pub is INF:
        return False
    w = pow(s, -1, c.n)
    u1 = e * w % c.n
    u2 = r * w % c.n
    R = ec_add(c, ec_mul(c, u1, c.G), ec_mul(c, u2, pub))
    if R is INF:
        return False
    return R[0] % c.n == r


# ---------------------------------------------------------------------------
# deterministic nonce source, protocol.cpp:13-34 and :67-75

def _splitmix(state: int):
    state = (state + 0x9E3779B97F4A7C15) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return state, z ^ (z >> 31)


def nonce(c: Curve, seed: int, stream: int, attempt: int = 0) -> int:
    state = seed & MASK64
    state, _ = _splitmix(state)
    state ^= (0xA3EC647659359ACD * (stream + 1)) & MASK64
    state, _ = _splitmix(state)
    state ^= (0xC2B2AE3D27D4EB4F * (attempt + 1)) & MASK64
    while True:
        raw = 0
        for i in range(4):  # w[2i] = lo32, w[2i+1] = hi32 -> 64-bit word i
            state, v = _splitmix(state)
            raw |= v << (64 * i)
        if 0 < raw < c.n:
            return raw


# ---------------------------------------------------------------------------
# wire codecs (sm2batch.h:4-9)

def be32(v: int) -> bytes:
    return v.to_bytes(32, "big")


def encode_point(pt) -> bytes:
    assert pt is not INF
    return b"\x04" + be32(pt[0]) + be32(pt[1])


def decode_point(c: Curve, rec: bytes):
    """curve.cpp:203-217 -- returns a point or raises ValueError."""
    if len(rec) != 65 or rec[0] != 4:
        raise ValueError("malformed")
    x = int.from_bytes(rec[1:33], "big")
    y = int.from_bytes(rec[33:65], "big")
    if x >= c.p or y >= c.p or not on_curve(c, (x, y)):
        raise ValueError("off curve")
    return (x, y)


def sign_lane(c: Curve, digest: bytes, secret: bytes, seed: int, stream: int):
    """One lane of sm2b_sign (capi.cpp:171-197 + protocol.cpp:106-168).
    Returns (64-byte signature, status)."""
    e = int.from_bytes(digest, "big")
    if e >= c.n:
        e -= c.n
    d = int.from_bytes(secret, "big")
    assert 0 < d < c.n
    for attempt in range(8):
        k = nonce(c, seed, stream, attempt)
        r, s = ecdsa_sign(c, e, d, k)
        if r == 0 or s == 0:
            continue
        return be32(r) + be32(s), 0
    return bytes(64), 5


def verify_lane(c: Curve, digest: bytes, pub: bytes, sig: bytes) -> int:
    """One lane of sm2b_verify (capi.cpp:199-228)."""
    e = int.from_bytes(digest, "big")
    if e >= c.n:
        e -= c.n
    try:
        Q = decode_point(c, pub)
    except ValueError:
        return 0
    r = int.from_bytes(sig[:32], "big")
    s = int.from_bytes(sig[32:], "big")
    return 1 if ecdsa_verify(c, e, Q, r, s) else 0


def msm(c: Curve, scalars, points):
    """sum_i scalars[i] * points[i]; definition only (no reference counterpart,
    SURVEY.md section 8c 'config 4')."""
    acc = INF
    for k, P in zip(scalars, points):
        acc = ec_add(c, acc, ec_mul(c, k % c.n, P))
    return acc
