#!/usr/bin/env python
"""Counts the field products our kernels execute per lane (verify / sign / keygen /
upmul) by running the product's own lane code on the host with instrumented
multiply / square / safegcd (tests/hostsim built with -DGECC_COUNT_OPS), at fixed-base
windows of 4 and 8 bits, and extrapolates linearly in the number of fixed-base
additions to the 16-bit window the GPU build uses.  Writes tools/op_counts.json,
which bench.py reads for its roofline arithmetic."""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from oracle import coracle as O  # noqa: E402

HS = os.path.join(ROOT, "tests", "hostsim")
KEYS = ["mul_generic", "mul_special", "sqr_generic", "sqr_special", "safegcd_generic", "safegcd_special"]


def run(wg, curve, n=256, hs_curve=None):
    hs_curve = curve if hs_curve is None else hs_curve
    lib = C.CDLL(os.path.join(HS, "_build", f"libgecc_hostsim_count{wg}.so"))
    p = lambda a: C.c_void_p(a.ctypes.data) if isinstance(a, np.ndarray) else C.cast(C.c_char_p(a), C.c_void_p)
    out = (C.c_ulonglong * 6)()
    rc, sec, pub = O.keygen(curve, 5, n)
    dig = np.random.RandomState(1).bytes(32 * n)
    rc, sig, st = O.ecdsa_sign(curve, dig, sec, 7)
    res = {}
    buf = lambda m: (C.c_uint8 * m)()
    lib.hs_keygen(hs_curve, C.c_size_t(1), C.c_uint64(1), C.c_uint64(0), buf(32), buf(65))  # builds the table
    lib.hs_op_counts(out, 1)
    s2, st2 = buf(64 * n), (C.c_int32 * n)()
    lib.hs_sign(hs_curve, C.c_size_t(n), p(dig), p(sec), C.c_uint64(7), C.c_uint64(0), s2, st2)
    assert bytes(s2) == sig
    lib.hs_op_counts(out, 1)
    res["sign"] = [v / n for v in out]
    r = buf(n)
    lib.hs_verify(hs_curve, C.c_size_t(n), p(dig), p(pub), p(sig), r)
    assert bytes(r) == b"\x01" * n
    lib.hs_op_counts(out, 1)
    res["verify"] = [v / n for v in out]
    lib.hs_keygen(hs_curve, C.c_size_t(n), C.c_uint64(9), C.c_uint64(0), buf(32 * n), buf(65 * n))
    lib.hs_op_counts(out, 1)
    res["keygen"] = [v / n for v in out]
    return res


def gadds(wg):  # expected fixed-base additions per scalar multiplication
    return (256 // wg) * (1 - 2.0 ** -wg) + 0.5 ** 1 * 0 + (0.5 if False else 0)


def main():
    subprocess.check_call(["make", "-C", HS, "count"], stdout=subprocess.DEVNULL)
    result = {}
    # the byte-record kernels run on the lazy curves (hostsim curve ids 2 and 3)
    for curve, name, hs in ((1, "secp256k1", 2), (0, "sm2", 3)):
        r4, r8 = run(4, curve, hs_curve=hs), run(8, curve, hs_curve=hs)
        ent = {}
        for op in r4:
            n4, n8, n16 = gadds(4), gadds(8), gadds(16)
            if op == "verify":
                pass  # one fixed-base multiplication per lane
            row = {}
            for i, k in enumerate(KEYS):
                slope = (r4[op][i] - r8[op][i]) / (n4 - n8)
                base = r8[op][i] - slope * n8
                row[k] = round(base + slope * n16, 2)
            ent[op] = row
        result[name] = ent
        print(name, json.dumps(ent, indent=1))
    with open(os.path.join(ROOT, "tools", "op_counts.json"), "w") as f:
        json.dump(result, f, indent=1)


if __name__ == "__main__":
    main()
