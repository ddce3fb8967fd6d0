#!/usr/bin/env python
"""Generates gecc_consts.cuh: per-field Montgomery constants and per-curve
parameters as constexpr accessors (folded to immediates after unrolling).

Everything here is derived from the four standard moduli with Python ints:
    q_inv32 = -q^-1 mod 2^32      (reference: FieldParams::make, field.cpp:166-170)
    r       = 2^256 mod q         (field.cpp:172-175)
    r2      = 2^512 mod q         (field.cpp:176-177)
    ninv    = -q^-1 mod 2^256     (full-width REDC constant used by the generic path)
Run:  python gen_consts.py > gecc_consts.cuh
"""
import sys

R = 1 << 256  # Montgomery radix of the 8-limb fields; an N-limb field uses 2^(32 N)


def limbs(v, n=8):
    return [(v >> (32 * i)) & 0xFFFFFFFF for i in range(n)]


def arr(v, n=8):
    return ", ".join("0x%08Xu" % w for w in limbs(v, n))


FIELDS = {
    "SecpP": 2**256 - 2**32 - 977,
    "SecpN": 0xFFFFFFFFFFFFFFFFFFFFFFFFFFFFFFFEBAAEDCE6AF48A03BBFD25E8CD0364141,
    "Sm2P": 2**256 - 2**224 - 2**96 + 2**64 - 1,
    "Sm2N": 0xFFFFFFFEFFFFFFFFFFFFFFFFFFFFFFFF7203DF6B21C6052B53BBF40939D54123,
    "SecpPL": 2**256 - 2**32 - 977,
    "Sm2PL": 2**256 - 2**224 - 2**96 + 2**64 - 1,
    # BLS12-381: 381-bit base field (12 limbs) and 255-bit scalar field (8 limbs)
    "Bls381P": 0x1a0111ea397fe69a4b1ba7b6434bacd764774b84f38512bf6730d2a0f6b0f6241eabfffeb153ffffb9feffffffffaaab,
    "Bls381R": 0x73eda753299d7d483339d80809a1d80553bda402fffe5bfeffffffff00000001,
    # BLS12-377: 377-bit base field (12 limbs) and 253-bit scalar field (8 limbs)
    "Bls377P": 0x01ae3a4617c510eac63b05c06ca1493b1a22d9f300f5138f1ef3622fba094800170b5d44300000008508c00000000001,
    "Bls377R": 0x12ab655e9a2ca55660b44d1e5c37b00159aa76fed00000010a11800000000001,
}
LIMBS = {"Bls381P": 12, "Bls377P": 12}
KIND = {"SecpP": "KIND_SECP_P", "SecpN": "KIND_GENERIC", "Sm2P": "KIND_SM2_P", "Sm2N": "KIND_GENERIC",
        "SecpPL": "KIND_SECP_LAZY", "Sm2PL": "KIND_SM2_LAZY", "Bls381P": "KIND_GENERIC", "Bls381R": "KIND_GENERIC",
        "Bls377P": "KIND_GENERIC", "Bls377R": "KIND_GENERIC"}
# SecpPL: the same prime as SecpP in a plain (non-Montgomery), weakly reduced representation
# used inside the fused ECDSA kernels: "R" is 1, elements live in [0, 2^256).
PLAIN = {"SecpPL"}
# Sm2PL: the SM2 prime in MONTGOMERY form (R = 2^256, the tables and constants of Sm2P serve), weakly
# reduced: any 256-bit value congruent to the element; used inside the fused ECDSA kernels.

CURVES = {
    "Secp": dict(fp="SecpP", fn="SecpN", a=0, b=7,
                 gx=0x79BE667EF9DCBBAC55A06295CE870B07029BFCDB2DCE28D959F2815B16F81798,
                 gy=0x483ADA7726A3C4655DA4FBFC0E1108A8FD17B448A68554199C47D08FFB10D4B8,
                 a_kind="A_ZERO"),
    "SecpL": dict(fp="SecpPL", fn="SecpN", a=0, b=7,
                  gx=0x79BE667EF9DCBBAC55A06295CE870B07029BFCDB2DCE28D959F2815B16F81798,
                  gy=0x483ADA7726A3C4655DA4FBFC0E1108A8FD17B448A68554199C47D08FFB10D4B8,
                  a_kind="A_ZERO"),
    "Sm2L": dict(fp="Sm2PL", fn="Sm2N", a=FIELDS["Sm2P"] - 3,
                 b=0x28E9FA9E9D9F5E344D5A9E4BCF6509A7F39789F515AB8F92DDBCBD414D940E93,
                 gx=0x32C4AE2C1F1981195F9904466A39C9948FE30BBFF2660BE1715A4589334C74C7,
                 gy=0xBC3736A2F4F6779C59BDCEE36B692153D0A9877CC62A474002DF32E52139F0A0,
                 a_kind="A_MINUS3"),
    "Sm2": dict(fp="Sm2P", fn="Sm2N", a=FIELDS["Sm2P"] - 3,
                b=0x28E9FA9E9D9F5E344D5A9E4BCF6509A7F39789F515AB8F92DDBCBD414D940E93,
                gx=0x32C4AE2C1F1981195F9904466A39C9948FE30BBFF2660BE1715A4589334C74C7,
                gy=0xBC3736A2F4F6779C59BDCEE36B692153D0A9877CC62A474002DF32E52139F0A0,
                a_kind="A_MINUS3"),
    # BLS12-381 G1: y^2 = x^3 + 4, the standard generator
    "Bls381": dict(fp="Bls381P", fn="Bls381R", a=0, b=4,
                   gx=0x17f1d3a73197d7942695638c4fa9ac0fc3688c4f9774b905a14e3a3f171bac586c55e83ff97a1aeffb3af00adb22c6bb,
                   gy=0x08b3f481e3aaa0f1a09e30ed741d8ae4fcf5e095d5d00af600db18cb2c04b3edd03cc744a2888ae40caa232946c5e7e1,
                   a_kind="A_ZERO"),
    # BLS12-377 G1: y^2 = x^3 + 1, the arkworks / Zexe generator (checked below: on the curve; its
    # order is the 253-bit r, checked in tests/test_hostsim_bls.py)
    "Bls377": dict(fp="Bls377P", fn="Bls377R", a=0, b=1,
                   gx=0x008848defe740a67c8fc6225bf87ff5485951e2caa9d41bb188282c8bd37cb5cd5481512ffcd394eeab9b16eb21be9ef,
                   gy=0x01914a69c5102eff1f674f5d30afeec4bd7fb348ca3e52d96d182ad44fb82305c2fe3d3634a9591afd82de55559c8ea6,
                   a_kind="A_ZERO"),
}
for _c in CURVES.values():
    _p = FIELDS[_c["fp"]]
    assert (_c["gy"] ** 2 - _c["gx"] ** 3 - _c["a"] * _c["gx"] - _c["b"]) % _p == 0


def table_fn(name, v, n=8):
    return ("    GECC_HD static constexpr uint32_t %s(int i) {\n"
            "        constexpr uint32_t t[%d] = {%s};\n        return t[i];\n    }\n" % (name, n, arr(v, n)))


def main():
    out = []
    w = out.append
    w("// GENERATED by gen_consts.py -- do not edit.\n#pragma once\n#include \"gecc_prims.cuh\"\n")
    w("namespace gecc {\n")
    w("enum FieldKind { KIND_GENERIC = 0, KIND_SECP_P = 1, KIND_SM2_P = 2, KIND_SECP_LAZY = 3, KIND_SM2_LAZY = 4 };")
    w("enum CurveA { A_ZERO = 0, A_MINUS3 = 1, A_GENERIC = 2 };\n")
    for name, q in FIELDS.items():
        nl = LIMBS.get(name, 8)
        R = 1 << (32 * nl)
        l30 = 9 if nl == 8 else (32 * nl + 29) // 30
        w("struct %s {" % name)
        w("    static constexpr int N = %d;" % nl)
        w("    static constexpr int kind = %s;" % KIND[name])
        w("    static constexpr uint32_t qinv32 = 0x%08Xu;  // -q^-1 mod 2^32" % ((-pow(q, -1, 1 << 32)) % (1 << 32)))
        Rf = 1 if name in PLAIN else R
        w(table_fn("q", q, nl))
        w(table_fn("r", Rf % q, nl))
        w(table_fn("r2", Rf * Rf % q, nl))
        w(table_fn("ninv", (-pow(q, -1, R)) % R, nl))
        w(table_fn("qm2", q - 2, nl))
        w(table_fn("r3", Rf * Rf * Rf % q, nl))
        # safegcd constants: q in 30-bit limbs and q^-1 mod 2^30
        w("    GECC_HD static constexpr uint32_t q30(int i) {\n        constexpr uint32_t t[%d] = {%s};\n        return t[i];\n    }"
          % (l30, ", ".join("0x%08Xu" % ((q >> (30 * i)) & 0x3FFFFFFF) for i in range(l30))))
        w("    GECC_HD static constexpr uint32_t qinv30() { return 0x%08Xu; }" % pow(q, -1, 1 << 30))
        w("};\n")
    for name, c in CURVES.items():
        p = FIELDS[c["fp"]]
        n = FIELDS[c["fn"]]
        nl = LIMBS.get(c["fp"], 8)
        Rc = 1 if c["fp"] in PLAIN else 1 << (32 * nl)
        m = lambda v: v * Rc % p
        w("struct %sCurve {" % name)
        w("    using Fp = %s;\n    using Fn = %s;" % (c["fp"], c["fn"]))
        w("    static constexpr int a_kind = %s;" % c["a_kind"])
        w("    static constexpr bool has_glv = %s;" % ("true" if name in ("Secp", "SecpL") else "false"))
        w(table_fn("a", m(c["a"]), nl))
        w(table_fn("b", m(c["b"]), nl))
        w(table_fn("gx", m(c["gx"]), nl))
        w(table_fn("gy", m(c["gy"]), nl))
        w(table_fn("three_b", m(3 * c["b"] % p), nl))
        if name in ("Secp", "SecpL"):
            # GLV endomorphism phi(x,y) = (beta*x, y) = lambda*(x,y); constants as in the
            # standard secp256k1 decomposition (Gallant-Lambert-Vanstone; values re-derived
            # and checked below: lambda^3 = 1 mod n, beta^3 = 1 mod p, lambda*G = (beta*Gx, Gy)).
            lam = 0x5363AD4CC05C30E0A5261C028812645A122E22EA20816678DF02967C1B23BD72
            beta = 0x7AE96A2B657C07106E64479EAC3434E99CF0497512F58995C1396C28719501EE
            assert pow(lam, 3, n) == 1 and pow(beta, 3, p) == 1
            a1 = 0x3086D221A7D46BCDE86C90E49284EB15
            b1 = -0xE4437ED6010E88286F547FA90ABFE4C3
            a2 = 0x114CA50F7A8E2F3F657C1108D9D44CFD8
            b2 = a1
            assert (a1 + b1 * lam) % n == 0 and (a2 + b2 * lam) % n == 0
            # rounding constants g1 = round(2^384 * b2 / n), g2 = round(2^384 * (-b1) / n)
            g1 = ((1 << 384) * b2 + n // 2) // n
            g2 = ((1 << 384) * (-b1) + n // 2) // n
            w(table_fn("beta", m(beta)))
            w(table_fn("lambda", lam))
            w(table_fn("glv_g1", g1))
            w(table_fn("glv_g2", g2))
            w(table_fn("glv_minus_b1", -b1, 4))
            w(table_fn("glv_b2", b2, 4))
            w(table_fn("glv_a1", a1, 4))
            w(table_fn("glv_a2", a2, 5))
        w("};\n")
    w("}  // namespace gecc")
    sys.stdout.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
