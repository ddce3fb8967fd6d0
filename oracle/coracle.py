"""TEST INFRASTRUCTURE ONLY -- ctypes view of oracle/_build/libgecc_oracle.so
(the plain-C restatement, oracle/gecc_oracle.c).  Same call shapes as
oracle/refshim.py so tests can run one against the other.
Only tests/, __graft_entry__.smoke() and bench.py's CPU arm may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .refshim import _p32, _p8, _buf, ints_to_cols, cols_to_ints, OPS  # noqa: F401

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libgecc_oracle.so")

_lib = None


def build():
    subprocess.check_call(["make", "-C", HERE, "oracle"], stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH, mode=os.RTLD_LOCAL)
        _lib.go_field_params.restype = C.c_uint32
    return _lib


def _check(rc, what):
    if rc:
        raise ValueError(f"{what} rc={rc}")


def field_params(curve, which):
    q, r, r2 = (np.zeros(8, np.uint32) for _ in range(3))
    qinv = lib().go_field_params(curve, which, _p32(q), _p32(r), _p32(r2))
    to_int = lambda a: int.from_bytes(a.astype("<u4").tobytes(), "little")
    return dict(q=to_int(q), q_inv=int(qinv), r=to_int(r), r2=to_int(r2))


def curve_params(curve):
    arrs = [np.zeros(8, np.uint32) for _ in range(4)]
    lib().go_curve_params(curve, *[_p32(a) for a in arrs])
    to_int = lambda a: int.from_bytes(a.astype("<u4").tobytes(), "little")
    return dict(zip(("a", "b", "gx", "gy"), map(to_int, arrs)))


def field_op(curve, which, op, a, b=None):
    n = a.shape[1]
    out = np.zeros((8, n), np.uint32)
    _check(lib().go_field_op(curve, which, OPS[op], C.c_size_t(n), _p32(a),
                             _p32(b) if b is not None else None, _p32(out)), "go_field_op")
    return out


def mont_reduce(curve, which, c16, sm2_route=False):
    n = c16.shape[1]
    out = np.zeros((8, n), np.uint32)
    _check(lib().go_mont_reduce(curve, which, int(sm2_route), C.c_size_t(n), _p32(c16),
                                _p32(out)), "go_mont_reduce")
    return out


def batch_invert(curve, which, a, lanes=0, workers=1):
    n = a.shape[1]
    out = np.zeros((8, n), np.uint32)
    _check(lib().go_batch_invert(curve, which, C.c_size_t(n), _p32(a), _p32(out),
                                 C.c_size_t(lanes)), "go_batch_invert")
    return out


def _pts_out(n):
    return (np.zeros((8, n), np.uint32), np.zeros((8, n), np.uint32), np.zeros(n, np.uint8))


def batch_padd(curve, P, T, lanes=0, workers=1):
    n = P[0].shape[1]
    ox, oy, oi = _pts_out(n)
    _check(lib().go_batch_padd(curve, C.c_size_t(n), _p32(P[0]), _p32(P[1]), _p8(P[2]),
                               _p32(T[0]), _p32(T[1]), _p8(T[2]), _p32(ox), _p32(oy), _p8(oi),
                               C.c_size_t(lanes)), "go_batch_padd")
    return ox, oy, oi


def batch_pdbl(curve, P, lanes=0, workers=1):
    n = P[0].shape[1]
    ox, oy, oi = _pts_out(n)
    _check(lib().go_batch_pdbl(curve, C.c_size_t(n), _p32(P[0]), _p32(P[1]), _p8(P[2]),
                               _p32(ox), _p32(oy), _p8(oi), C.c_size_t(lanes)), "go_batch_pdbl")
    return ox, oy, oi


def batch_fpmul(curve, scalars, lanes=0, workers=1):
    n = scalars.shape[1]
    ox, oy, oi = _pts_out(n)
    _check(lib().go_batch_fpmul(curve, C.c_size_t(n), _p32(scalars), _p32(ox), _p32(oy),
                                _p8(oi), C.c_size_t(lanes)), "go_batch_fpmul")
    return ox, oy, oi


def batch_upmul(curve, scalars, P, lanes=0, workers=1):
    n = scalars.shape[1]
    ox, oy, oi = _pts_out(n)
    _check(lib().go_batch_upmul(curve, C.c_size_t(n), _p32(scalars), _p32(P[0]), _p32(P[1]),
                                _p8(P[2]), _p32(ox), _p32(oy), _p8(oi), C.c_size_t(lanes)),
           "go_batch_upmul")
    return ox, oy, oi


def pmul_serial(curve, scalars, P):
    n = scalars.shape[1]
    ox, oy, oi = _pts_out(n)
    _check(lib().go_pmul_serial(curve, C.c_size_t(n), _p32(scalars), _p32(P[0]), _p32(P[1]),
                                _p8(P[2]), _p32(ox), _p32(oy), _p8(oi)), "go_pmul_serial")
    return ox, oy, oi


def msm(curve, scalars, P):
    n = scalars.shape[1]
    ox, oy, oi = _pts_out(1)
    _check(lib().go_msm(curve, C.c_size_t(n), _p32(scalars), _p32(P[0]), _p32(P[1]), _p8(P[2]),
                        _p32(ox), _p32(oy), _p8(oi)), "go_msm")
    return ox, oy, oi


def nonce(curve, seed, stream, attempt=0) -> int:
    out = (C.c_uint8 * 32)()
    lib().go_nonce(curve, C.c_uint64(seed), C.c_uint64(stream), C.c_uint32(attempt), out)
    return int.from_bytes(bytes(out), "big")


def keygen(curve, seed, count, lane_base=0, lanes=0, workers=1):
    sec = (C.c_uint8 * (32 * count))()
    pub = (C.c_uint8 * (65 * count))()
    rc = lib().go_keygen(curve, C.c_uint64(seed), C.c_uint64(lane_base), C.c_size_t(count),
                         sec, pub, C.c_size_t(lanes))
    return rc, bytes(sec), bytes(pub)


def ecdsa_sign(curve, digests, secrets, seed, lane_base=0, lanes=0, workers=1, want_status=True):
    count = len(digests) // 32
    sig = (C.c_uint8 * (64 * count))()
    st = (C.c_int32 * count)() if want_status else None
    rc = lib().go_sign(curve, C.c_size_t(count), _buf(digests), _buf(secrets), C.c_uint64(seed),
                       C.c_uint64(lane_base), sig, st, C.c_size_t(lanes))
    return rc, bytes(sig), (list(st) if st is not None else None)


def ecdsa_verify(curve, digests, publics, sigs, lanes=0, workers=1):
    count = len(digests) // 32
    res = (C.c_uint8 * count)()
    rc = lib().go_verify(curve, C.c_size_t(count), _buf(digests), _buf(publics), _buf(sigs),
                         res, C.c_size_t(lanes))
    return rc, bytes(res)


def ecdh(curve, secrets, peers, lanes=0, workers=1, want_status=True):
    count = len(secrets) // 32
    sh = (C.c_uint8 * (32 * count))()
    st = (C.c_int32 * count)() if want_status else None
    rc = lib().go_ecdh(curve, C.c_size_t(count), _buf(secrets), _buf(peers), sh, st,
                       C.c_size_t(lanes))
    return rc, bytes(sh), (list(st) if st is not None else None)


def ledger():
    arr = (C.c_uint64 * 4)()
    lib().go_ledger_read(arr)
    return dict(zip(("modmul", "modadd", "modsub", "modinv"), list(arr)))


def ledger_reset():
    lib().go_ledger_reset()
