"""TEST INFRASTRUCTURE ONLY -- ctypes view of oracle/_ref/libgecc_ref.so.

That library is the UNMODIFIED reference (compiled from /root/reference/proj/src
by oracle/Makefile) plus oracle/ref_shim.cpp.  It is the strongest checker we
have: the real reference kernels, run here or on the GPU box's host cores.
Only tests/, __graft_entry__.smoke() and bench.py's CPU arm may import this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libgecc_ref.so")

_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)
_i32p = C.POINTER(C.c_int32)


def available() -> bool:
    return os.path.exists(LIB_PATH)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(
                "oracle/_ref/libgecc_ref.so missing: run `make -C oracle ref` where "
                "/root/reference exists")
        _lib = C.CDLL(LIB_PATH, mode=os.RTLD_LOCAL)
        _lib.ref_field_params.restype = C.c_uint32
        _lib.sm2b_ctx_new.restype = C.c_void_p
        _lib.sm2b_ctx_free.argtypes = [C.c_void_p]
        _lib.sm2b_version.restype = C.c_char_p
    return _lib


# --- numpy <-> int helpers (column-major limbs: arr[k, i] = limb k of element i)

def ints_to_cols(vals) -> np.ndarray:
    n = len(vals)
    raw = b"".join(int(v).to_bytes(32, "little") for v in vals)
    return np.ascontiguousarray(np.frombuffer(raw, dtype="<u4").reshape(n, 8).T)


def cols_to_ints(cols: np.ndarray):
    rows = np.ascontiguousarray(cols.T).astype("<u4")
    return [int.from_bytes(rows[i].tobytes(), "little") for i in range(rows.shape[0])]


def _p32(a):
    return a.ctypes.data_as(_u32p)


def _p8(a):
    return a.ctypes.data_as(_u8p) if a is not None else None


def field_params(curve: int, which: int):
    q = np.zeros(8, np.uint32)
    r = np.zeros(8, np.uint32)
    r2 = np.zeros(8, np.uint32)
    qinv = lib().ref_field_params(curve, which, _p32(q), _p32(r), _p32(r2))
    to_int = lambda a: int.from_bytes(a.astype("<u4").tobytes(), "little")
    return dict(q=to_int(q), q_inv=int(qinv), r=to_int(r), r2=to_int(r2))


def curve_params(curve: int):
    arrs = [np.zeros(8, np.uint32) for _ in range(4)]
    lib().ref_curve_params(curve, *[_p32(a) for a in arrs])
    to_int = lambda a: int.from_bytes(a.astype("<u4").tobytes(), "little")
    return dict(zip(("a", "b", "gx", "gy"), map(to_int, arrs)))


OPS = dict(mont_mul=0, mod_add=1, mod_sub=2, to_mont=3, from_mont=4, mod_inv=5)


def field_op(curve: int, which: int, op: str, a: np.ndarray, b: np.ndarray | None = None):
    n = a.shape[1]
    out = np.zeros((8, n), np.uint32)
    rc = lib().ref_field_op(curve, which, OPS[op], C.c_size_t(n), _p32(a),
                            _p32(b) if b is not None else None, _p32(out))
    if rc:
        raise ValueError(f"ref_field_op rc={rc}")
    return out


def mont_reduce(curve: int, which: int, c16: np.ndarray, sm2_route: bool = False):
    n = c16.shape[1]
    out = np.zeros((8, n), np.uint32)
    rc = lib().ref_mont_reduce(curve, which, int(sm2_route), C.c_size_t(n), _p32(c16), _p32(out))
    if rc:
        raise ValueError(f"ref_mont_reduce rc={rc}")
    return out


def batch_invert(curve, which, a, lanes=0, workers=1):
    n = a.shape[1]
    out = np.zeros((8, n), np.uint32)
    rc = lib().ref_batch_invert(curve, which, C.c_size_t(n), _p32(a), _p32(out),
                                C.c_size_t(lanes), workers)
    if rc:
        raise ValueError(f"ref_batch_invert rc={rc}")
    return out


def _pts_out(n):
    return (np.zeros((8, n), np.uint32), np.zeros((8, n), np.uint32), np.zeros(n, np.uint8))


def batch_padd(curve, P, T, lanes=0, workers=1):
    """P, T = (x_cols, y_cols, inf_u8) in Montgomery form."""
    n = P[0].shape[1]
    ox, oy, oi = _pts_out(n)
    rc = lib().ref_batch_padd(curve, C.c_size_t(n), _p32(P[0]), _p32(P[1]), _p8(P[2]),
                              _p32(T[0]), _p32(T[1]), _p8(T[2]), _p32(ox), _p32(oy), _p8(oi),
                              C.c_size_t(lanes), workers)
    if rc:
        raise ValueError(f"ref_batch_padd rc={rc}")
    return ox, oy, oi


def batch_padd_timed(curve, P, T, lanes=0, workers=0, repeats=5) -> float:
    n = P[0].shape[1]
    secs = C.c_double(0)
    rc = lib().ref_batch_padd_timed(curve, C.c_size_t(n), _p32(P[0]), _p32(P[1]), _p32(T[0]),
                                    _p32(T[1]), C.c_size_t(lanes), workers, repeats,
                                    C.byref(secs))
    if rc:
        raise ValueError(f"ref_batch_padd_timed rc={rc}")
    return secs.value


def batch_pdbl(curve, P, lanes=0, workers=1):
    n = P[0].shape[1]
    ox, oy, oi = _pts_out(n)
    rc = lib().ref_batch_pdbl(curve, C.c_size_t(n), _p32(P[0]), _p32(P[1]), _p8(P[2]),
                              _p32(ox), _p32(oy), _p8(oi), C.c_size_t(lanes), workers)
    if rc:
        raise ValueError(f"ref_batch_pdbl rc={rc}")
    return ox, oy, oi


def batch_fpmul(curve, scalars, lanes=0, workers=1):
    n = scalars.shape[1]
    ox, oy, oi = _pts_out(n)
    rc = lib().ref_batch_fpmul(curve, C.c_size_t(n), _p32(scalars), _p32(ox), _p32(oy), _p8(oi),
                               C.c_size_t(lanes), workers)
    if rc:
        raise ValueError(f"ref_batch_fpmul rc={rc}")
    return ox, oy, oi


def batch_upmul(curve, scalars, P, lanes=0, workers=1):
    n = scalars.shape[1]
    ox, oy, oi = _pts_out(n)
    rc = lib().ref_batch_upmul(curve, C.c_size_t(n), _p32(scalars), _p32(P[0]), _p32(P[1]),
                               _p8(P[2]), _p32(ox), _p32(oy), _p8(oi), C.c_size_t(lanes), workers)
    if rc:
        raise ValueError(f"ref_batch_upmul rc={rc}")
    return ox, oy, oi


def pmul_serial(curve, scalars, P):
    n = scalars.shape[1]
    ox, oy, oi = _pts_out(n)
    rc = lib().ref_pmul_serial(curve, C.c_size_t(n), _p32(scalars), _p32(P[0]), _p32(P[1]),
                               _p8(P[2]), _p32(ox), _p32(oy), _p8(oi))
    if rc:
        raise ValueError(f"ref_pmul_serial rc={rc}")
    return ox, oy, oi


def nonce(curve, seed, stream, attempt=0) -> int:
    out = (C.c_uint8 * 32)()
    lib().ref_nonce(curve, C.c_uint64(seed), C.c_uint64(stream), C.c_uint32(attempt), out)
    return int.from_bytes(bytes(out), "big")


def _buf(b: bytes):
    return (C.c_uint8 * len(b)).from_buffer_copy(b) if len(b) else None


def keygen(curve, seed, count, lane_base=0, lanes=0, workers=1):
    sec = (C.c_uint8 * (32 * count))()
    pub = (C.c_uint8 * (65 * count))()
    rc = lib().ref_keygen(curve, C.c_uint64(seed), C.c_uint64(lane_base), C.c_size_t(count),
                          sec, pub, C.c_size_t(lanes), workers)
    return rc, bytes(sec), bytes(pub)


def ecdsa_sign(curve, digests: bytes, secrets: bytes, seed, lane_base=0, lanes=0, workers=1,
               want_status=True):
    count = len(digests) // 32
    sig = (C.c_uint8 * (64 * count))()
    st = (C.c_int32 * count)() if want_status else None
    rc = lib().ref_ecdsa_sign(curve, C.c_size_t(count), _buf(digests), _buf(secrets),
                              C.c_uint64(seed), C.c_uint64(lane_base), sig, st,
                              C.c_size_t(lanes), workers)
    return rc, bytes(sig), (list(st) if st is not None else None)


def ecdsa_verify(curve, digests: bytes, publics: bytes, sigs: bytes, lanes=0, workers=1):
    count = len(digests) // 32
    res = (C.c_uint8 * count)()
    rc = lib().ref_ecdsa_verify(curve, C.c_size_t(count), _buf(digests), _buf(publics),
                                _buf(sigs), res, C.c_size_t(lanes), workers)
    return rc, bytes(res)


def ecdh(curve, secrets: bytes, peers: bytes, lanes=0, workers=1, want_status=True):
    count = len(secrets) // 32
    sh = (C.c_uint8 * (32 * count))()
    st = (C.c_int32 * count)() if want_status else None
    rc = lib().ref_ecdh(curve, C.c_size_t(count), _buf(secrets), _buf(peers), sh, st,
                        C.c_size_t(lanes), workers)
    return rc, bytes(sh), (list(st) if st is not None else None)


class Sm2bCtx:
    """The reference's own C ABI (sm2batch.h:44-105), SM2 only."""

    def __init__(self, workers=1, lanes=0):
        self.l = lib()
        self.ctx = C.c_void_p(self.l.sm2b_ctx_new(workers, lanes))
        assert self.ctx.value

    def close(self):
        if self.ctx:
            self.l.sm2b_ctx_free(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def keygen(self, seed, count):
        sec = (C.c_uint8 * (32 * count))()
        pub = (C.c_uint8 * (65 * count))()
        rc = self.l.sm2b_keygen(self.ctx, C.c_uint64(seed), C.c_size_t(count), sec, pub)
        return rc, bytes(sec), bytes(pub)

    def sign(self, digests, secrets, seed, want_status=True):
        count = len(digests) // 32
        sig = (C.c_uint8 * (64 * count))()
        st = (C.c_int32 * count)() if want_status else None
        rc = self.l.sm2b_sign(self.ctx, C.c_size_t(count), _buf(digests), _buf(secrets),
                              C.c_uint64(seed), sig, st)
        return rc, bytes(sig), (list(st) if st is not None else None)

    def verify(self, digests, publics, sigs):
        count = len(digests) // 32
        res = (C.c_uint8 * count)()
        rc = self.l.sm2b_verify(self.ctx, C.c_size_t(count), _buf(digests), _buf(publics),
                                _buf(sigs), res)
        return rc, bytes(res)

    def ecdh(self, secrets, peers, want_status=True):
        count = len(secrets) // 32
        sh = (C.c_uint8 * (32 * count))()
        st = (C.c_int32 * count)() if want_status else None
        rc = self.l.sm2b_ecdh(self.ctx, C.c_size_t(count), _buf(secrets), _buf(peers), sh, st)
        return rc, bytes(sh), (list(st) if st is not None else None)

    def ledger(self):
        arr = (C.c_uint64 * 4)()
        self.l.sm2b_ledger_read(self.ctx, arr)
        return dict(zip(("modmul", "modadd", "modsub", "modinv"), list(arr)))

    def ledger_reset(self):
        self.l.sm2b_ledger_reset(self.ctx)
