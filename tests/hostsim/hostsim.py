"""TEST-ONLY ctypes view of tests/hostsim/_build/libgecc_hostsim.so: the product's
__host__ __device__ limb / curve / ECDSA-lane code compiled for the CPU."""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libgecc_hostsim.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        subprocess.check_call(["make", "-C", HERE], stdout=subprocess.DEVNULL)
        _lib = C.CDLL(LIB, mode=os.RTLD_LOCAL)
    return _lib


def _p(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.cast(C.c_char_p(bytes(a)), C.c_void_p) if len(a) else None


FIELD_IDS = {(1, 0): 0, (1, 1): 1, (0, 0): 2, (0, 1): 3}  # (curve, which) -> hostsim field id
OPS = dict(mont_mul=0, mod_add=1, mod_sub=2, to_mont=3, from_mont=4, mod_inv=5, sqr=6, inv_safegcd=7, inv_plain=8, dbl=9, mul8=10, inv_var=11, inv_var_plain=12, inv_sched_plain=13, inv_sched_exit_plain=14)


SECP_LAZY_CURVE = 2   # secp256k1 in the lazy plain representation (ECDSA kernels)
SECP_LAZY_FIELD = 5
SM2_LAZY_CURVE = 3    # SM2 in weakly reduced Montgomery form (ECDSA kernels)
SM2_LAZY_FIELD = 10


BLS_P_FIELD, BLS_R_FIELD = 6, 7   # BLS12-381 base field (12 limbs) and scalar field (8 limbs)
BLS_FIELDS = {2: (6, 7), 3: (8, 9)}  # curve id -> (base field, scalar field) hostsim ids; 3 = BLS12-377


def field_op(curve, which, op, a, b=None, field_id=None):
    n = a.shape[1]
    out = np.zeros((a.shape[0], n), np.uint32)
    fid = FIELD_IDS[(curve, which)] if field_id is None else field_id
    rc = lib().hs_field_op(fid, None, OPS[op], C.c_size_t(n), _p(a), _p(b), _p(out))
    assert rc == 0
    return out


def _pts(n):
    return np.zeros((8, n), np.uint32), np.zeros((8, n), np.uint32), np.zeros(n, np.uint8)


def batch_fpmul(curve, k):
    n = k.shape[1]
    o = _pts(n)
    assert lib().hs_fpmul(curve, C.c_size_t(n), _p(k), _p(o[0]), _p(o[1]), _p(o[2])) == 0
    return o


def batch_upmul(curve, k, P):
    n = k.shape[1]
    o = _pts(n)
    assert lib().hs_upmul(curve, C.c_size_t(n), _p(k), _p(P[0]), _p(P[1]), _p(P[2]), _p(o[0]),
                          _p(o[1]), _p(o[2])) == 0
    return o


def slot_adds(curve, P, Q, lam):
    """0 when every slot-form addition agrees with jac_madd on the pairs (P_i, Q_i); see hs_slot_adds."""
    n = P[0].shape[1]
    return lib().hs_slot_adds(curve, C.c_size_t(n), _p(P[0]), _p(P[1]), _p(Q[0]), _p(Q[1]), _p(lam))


def sign(curve, dig, sec, seed, lane_base=0):
    n = len(dig) // 32
    sig = (C.c_uint8 * max(1, 64 * n))()
    st = (C.c_int32 * max(1, n))()
    assert lib().hs_sign(curve, C.c_size_t(n), _p(dig), _p(sec), C.c_uint64(seed),
                         C.c_uint64(lane_base), sig, st) == 0
    return bytes(sig)[:64 * n], list(st)[:n]


def verify(curve, dig, pub, sig):
    n = len(dig) // 32
    res = (C.c_uint8 * max(1, n))()
    assert lib().hs_verify(curve, C.c_size_t(n), _p(dig), _p(pub), _p(sig), res) == 0
    return bytes(res)[:n]


def keygen(curve, seed, n, lane_base=0):
    sec = (C.c_uint8 * max(1, 32 * n))()
    pub = (C.c_uint8 * max(1, 65 * n))()
    assert lib().hs_keygen(curve, C.c_size_t(n), C.c_uint64(seed), C.c_uint64(lane_base), sec, pub) == 0
    return bytes(sec)[:32 * n], bytes(pub)[:65 * n]


def redc(curve, which, c16):
    n = c16.shape[1]
    out = np.zeros((8, n), np.uint32)
    assert lib().hs_redc(FIELD_IDS[(curve, which)], C.c_size_t(n), _p(c16), _p(out)) == 0
    return out


def glv_split(k):
    n = k.shape[1]
    m1, m2, sg = np.zeros((8, n), np.uint32), np.zeros((8, n), np.uint32), np.zeros(2 * n, np.uint8)
    assert lib().hs_glv_split(C.c_size_t(n), _p(k), _p(m1), _p(m2), _p(sg)) == 0
    return m1, m2, sg


def bls_point_op(op, P, T=None, k=None, curve=2):
    """BLS12-381 / BLS12-377 G1 (12-limb Montgomery coordinates): op 'add' | 'dbl' | 'mul'."""
    n = P[0].shape[1]
    o = np.zeros((12, n), np.uint32), np.zeros((12, n), np.uint32), np.zeros(n, np.uint8)
    T = T if T is not None else P
    rc = lib().hs_bls_point_op(curve, {"add": 0, "dbl": 1, "mul": 2}[op], C.c_size_t(n), _p(k), _p(P[0]), _p(P[1]),
                               _p(P[2]), _p(T[0]), _p(T[1]), _p(T[2]), _p(o[0]), _p(o[1]), _p(o[2]))
    assert rc == 0, rc
    return o


def set_uniform(on: bool):
    """Selects the constant-structure forms (GECC_SECRET_UNIFORM) of k*G, k*P, sign and keygen."""
    lib().hs_set_uniform(1 if on else 0)


def sign_nonces(curve, dig, sec, nonces):
    n = len(dig) // 32
    sig = (C.c_uint8 * max(1, 64 * n))()
    st = (C.c_int32 * max(1, n))()
    assert lib().hs_sign_nonces(curve, C.c_size_t(n), _p(dig), _p(sec), _p(nonces), sig, st) == 0
    return bytes(sig)[:64 * n], list(st)[:n]
