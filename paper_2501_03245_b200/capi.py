"""ctypes binding of include/gecc_b200.h.

Method names and argument meaning mirror the reference's interface for this path
(sm2batch.h: keygen / sign / verify / ecdh; batch_point.hpp: batch_padd / batch_pdbl /
batch_fpmul / batch_upmul; batch_invert.hpp: batch_invert) so that the parity tests
read like the reference's own tests.  Column buffers are numpy uint32 arrays of shape
(8, n): arr[k, i] = limb k of element i (batch_buffer.hpp:15-35).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# GECC_LIB selects an experiment build of the same library (csrc/Makefile VARIANT=...), for A/B timing
LIB_PATH = os.environ.get("GECC_LIB") or os.path.join(HERE, "lib", "libgecc_b200.so")

SM2, SECP256K1, BLS12_381, BLS12_377 = 0, 1, 2, 3
FIELD_P, FIELD_N = 0, 1
STATUS = {0: "ok", 1: "invalid argument", 2: "malformed input", 3: "invalid peer point",
          4: "degenerate result", 5: "nonce retries exhausted", 6: "cost model has no crossover",
          7: "internal error"}
FIELD_OPS = dict(mont_mul=0, mod_add=1, mod_sub=2, to_mont=3, from_mont=4, mod_inv=5, mod_inv_fermat=6,
                 mont_reduce=7, lazy_mul=8, lazy_sqr=9, lazy_add=10, lazy_sub=11, mod_inv_warp=12)
SECRET_FAST, SECRET_UNIFORM = 0, 1
COMM_ID_BYTES = 128


class GeccError(RuntimeError):
    pass


_lib = None


def lib_available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    """Loads libgecc_b200.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not lib_available():
            raise GeccError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; "
                            "g.build()'` or `make -C paper_2501_03245_b200/csrc`")
        l = C.CDLL(LIB_PATH, mode=os.RTLD_LOCAL)
        l.sm2b_ctx_new.restype = C.c_void_p
        l.sm2b_ctx_new.argtypes = [C.c_uint32, C.c_uint32]
        l.gecc_ctx_new.restype = C.c_void_p
        l.gecc_ctx_new.argtypes = [C.c_int, C.c_int]
        l.gecc_ctx_new_multi.restype = C.c_void_p
        l.gecc_ctx_new_multi.argtypes = [C.c_int, C.c_int, C.c_void_p]
        l.gecc_ctx_shards.argtypes = [C.c_void_p]
        l.gecc_ctx_set_secret_mode.argtypes = [C.c_void_p, C.c_int]
        l.gecc_base_table_new.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        l.gecc_base_table_free.argtypes = [C.c_void_p]
        l.gecc_base_table_free.restype = None
        l.gecc_comm_unique_id.argtypes = [C.c_void_p]
        l.gecc_comm_init_rank.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        l.gecc_msm_combine_dev.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        l.sm2b_ctx_free.argtypes = [C.c_void_p]
        l.sm2b_version.restype = C.c_char_p
        l.sm2b_status_str.restype = C.c_char_p
        l.gecc_last_error.restype = C.c_char_p
        l.gecc_last_error.argtypes = [C.c_void_p]
        l.gecc_kernel_launches.restype = C.c_uint64
        l.gecc_kernel_launches.argtypes = [C.c_void_p]
        l.gecc_field_params_make.argtypes = [C.c_void_p, C.c_void_p]
        l.gecc_field_params_get.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        l.gecc_field_op_rt.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
        l.gecc_batch_invert_rt.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
        l.gecc_batch_padd_rt.argtypes = [C.c_void_p] * 3 + [C.c_size_t] + [C.c_void_p] * 9
        l.gecc_batch_pdbl_rt.argtypes = [C.c_void_p] * 3 + [C.c_size_t] + [C.c_void_p] * 6
        l.gecc_set_batch_form.argtypes = [C.c_int]
        l.gecc_set_batch_form.restype = None
        l.gecc_set_msm_form.argtypes = [C.c_int]
        l.gecc_set_msm_form.restype = None
        # A/B timing knobs (tools/, bench.py): pin a kernel form for the whole process
        if os.environ.get("GECC_MSM_FORM"):
            l.gecc_set_msm_form(int(os.environ["GECC_MSM_FORM"]))
        if os.environ.get("GECC_BATCH_FORM"):
            l.gecc_set_batch_form(int(os.environ["GECC_BATCH_FORM"]))
        _lib = l
    return _lib


BATCH_FORMS = {"auto": 0, "chunked": 1, "coop": 2, "chunked8": 3, "coop128": 4, "coop32": 5, "tiled8": 6, "tiled4": 7,
               "fused": 8, "fused2": 9}


def set_batch_form(form: str):
    """Pins the batch kernels' form (gecc_set_batch_form): auto | chunked | coop."""
    lib().gecc_set_batch_form(BATCH_FORMS[form])


MSM_FORMS = {"auto": 0, "jacobian": 1, "affine": 2, "affine1": 3, "fused16": 4, "fused8": 5}


def set_msm_form(form: str):
    """Pins gecc_msm's bucket accumulation (gecc_set_msm_form): auto | jacobian | affine."""
    lib().gecc_set_msm_form(MSM_FORMS[form])


def field_params_make(q: int):
    """FieldParams::make(q) (gecc_field_params_make): the opaque parameter block for the *_rt entry
    points, or ValueError for an even / too small modulus (no GPU needed)."""
    qa = np.frombuffer(int(q).to_bytes(32, "little"), np.uint32).copy()
    out = np.zeros(64, np.uint32)
    rc = lib().gecc_field_params_make(qa.ctypes.data, out.ctypes.data)
    if rc != 0:
        raise ValueError(f"gecc_field_params_make rc={rc}")
    return out


def field_params_get(params, which: int) -> int:
    """0 q, 1 R, 2 R^2, 3 R^3 of a parameter block"""
    out = np.zeros(8, np.uint32)
    rc = lib().gecc_field_params_get(params.ctypes.data, which, out.ctypes.data)
    if rc != 0:
        raise ValueError(f"gecc_field_params_get rc={rc}")
    return int.from_bytes(out.tobytes(), "little")


def cols_from_ints(vals, limbs: int = 8) -> np.ndarray:
    """ints -> column buffer [limbs, n] (limb k of element i at [k, i]; 8 limbs = 256 bits,
    12 limbs = the 381-bit coordinates of BLS12-381)"""
    n = len(vals)
    raw = b"".join(int(v).to_bytes(4 * limbs, "little") for v in vals)
    return np.ascontiguousarray(np.frombuffer(raw, dtype="<u4").reshape(n, limbs).T)


def ints_from_cols(cols: np.ndarray):
    rows = np.ascontiguousarray(cols.T).astype("<u4")
    return [int.from_bytes(rows[i].tobytes(), "little") for i in range(rows.shape[0])]


def _vp(a):
    """numpy array / bytes / int (raw address) / None -> void pointer argument"""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("buffer must be C-contiguous")
        return C.c_void_p(a.ctypes.data)
    if isinstance(a, (bytes, bytearray)):
        return C.cast(C.c_char_p(bytes(a)), C.c_void_p) if len(a) else None
    return C.c_void_p(int(a))


def _need_cols(a, rows, n, what):
    """column buffers are uint32 arrays of shape (rows, n): a short or mistyped buffer would make
    the C side read past the end of the Python object"""
    if not isinstance(a, np.ndarray) or a.dtype != np.uint32 or a.shape != (rows, n) or not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{what}: expected a C-contiguous uint32 array of shape ({rows}, {n})")


def _need_mask(a, n, what):
    if a is None:
        return
    if not isinstance(a, np.ndarray) or a.dtype != np.uint8 or a.shape != (n,) or not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{what}: expected a C-contiguous uint8 array of shape ({n},)")


def _need_bytes(b, size, what):
    if len(b) != size:
        raise ValueError(f"{what}: expected {size} bytes, got {len(b)}")


class BaseTable:
    """precompute_base_table(c, g) for an arbitrary on-curve g (batch_point.hpp:76-83): a device
    table owned by a Context; raises ValueError for an off-curve point as the reference throws
    std::invalid_argument (batch_point.cpp:343-344)."""

    def __init__(self, ctx: "Context", x: np.ndarray, y: np.ndarray):
        x = np.ascontiguousarray(x, np.uint32).reshape(8)
        y = np.ascontiguousarray(y, np.uint32).reshape(8)
        h = C.c_void_p()
        rc = ctx.l.gecc_base_table_new(ctx.h, _vp(x), _vp(y), C.byref(h))
        ctx._check(rc, "gecc_base_table_new")
        if rc != 0:
            raise ValueError("precompute_base_table: point off curve" if rc == 2 else f"gecc_base_table_new rc={rc}")
        self.ctx, self.h = ctx, h

    def close(self):
        if getattr(self, "h", None) and self.ctx.h:
            self.ctx.l.gecc_base_table_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0 draws it, the launcher broadcasts it)."""
    buf = (C.c_uint8 * COMM_ID_BYTES)()
    rc = lib().gecc_comm_unique_id(buf)
    if rc != 0:
        raise GeccError("gecc_comm_unique_id failed: libnccl.so.2 could not be loaded")
    return bytes(buf)


class Context:
    """One engine context = one curve on one CUDA device, or -- with ``devices`` -- a GROUP
    context that shards every host call over several devices (sm2b_ctx, sm2batch.h:41-45)."""

    def __init__(self, curve: int = SM2, device: int = -1, reference_compat: bool = False,
                 workers: int = 0, lanes: int = 0, devices=None):
        self.l = lib()
        if reference_compat:
            h = self.l.sm2b_ctx_new(workers, lanes)
        elif devices is not None:
            devs = np.ascontiguousarray(devices, np.int32)
            h = self.l.gecc_ctx_new_multi(curve, len(devs), _vp(devs) if len(devs) else None)
        else:
            h = self.l.gecc_ctx_new(curve, device)
        if not h:
            raise GeccError("gecc_ctx_new failed: no usable CUDA device or bad arguments "
                            "(libgecc_b200 has no CPU path)")
        self.h = C.c_void_p(h)
        self.curve = self.l.gecc_ctx_curve(self.h)
        self.limbs = 12 if self.curve in (BLS12_381, BLS12_377) else 8  # 32-bit limbs per coordinate

    def close(self):
        if getattr(self, "h", None):
            self.l.sm2b_ctx_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- plumbing
    def _check(self, rc, what):
        if rc == 7:
            raise GeccError(f"{what}: {self.l.gecc_last_error(self.h).decode()}")
        return rc

    @property
    def launches(self) -> int:
        return int(self.l.gecc_kernel_launches(self.h))

    def set_stream(self, stream_ptr: int | None):
        """None -> the context's own stream; 0 -> the CUDA legacy default stream
        (cudaStreamLegacy), anything else is taken as a cudaStream_t."""
        if stream_ptr is None:
            ptr = 0
        else:
            ptr = 1 if int(stream_ptr) == 0 else int(stream_ptr)  # 0x1 == cudaStreamLegacy
        self.l.gecc_ctx_set_stream(self.h, C.c_void_p(ptr))

    @property
    def shards(self) -> int:
        return int(self.l.gecc_ctx_shards(self.h))

    def set_secret_mode(self, mode: int):
        """SECRET_FAST | SECRET_UNIFORM (constant-structure k*G and d*P on secret scalars)."""
        if self.l.gecc_ctx_set_secret_mode(self.h, mode) != 0:
            raise ValueError("gecc_ctx_set_secret_mode: bad mode")

    def comm_init_rank(self, nranks: int, rank: int, unique_id: bytes):
        """Joins the multi-process MSM exchange communicator (ncclCommInitRank)."""
        _need_bytes(unique_id, COMM_ID_BYTES, "unique_id")
        rc = self.l.gecc_comm_init_rank(self.h, nranks, rank, _vp(unique_id))
        self._check(rc, "gecc_comm_init_rank")
        if rc != 0:
            raise ValueError(f"gecc_comm_init_rank rc={rc}")

    def ledger(self):
        arr = (C.c_uint64 * 4)()
        self.l.sm2b_ledger_read(self.h, arr)
        return dict(zip(("modmul", "modadd", "modsub", "modinv"), list(arr)))

    def ledger_reset(self):
        self.l.sm2b_ledger_reset(self.h)

    # -- field layer
    def field_op(self, field: int, op: str, a: np.ndarray, b: np.ndarray | None = None):
        n = a.shape[1]
        rows = self.limbs if field == 0 else 8
        _need_cols(a, rows, n, "field_op a")
        if b is not None:
            _need_cols(b, rows, n, "field_op b")
        out = np.zeros((rows, n), np.uint32)
        rc = self.l.gecc_field_op(self.h, field, FIELD_OPS[op], C.c_size_t(n), _vp(a), _vp(b), _vp(out))
        if self._check(rc, "gecc_field_op"):
            raise ValueError(f"gecc_field_op rc={rc}")
        return out

    def microbench(self, which: int, iters: int = 2000):
        r, s, t = C.c_double(), C.c_double(), C.c_double()
        rc = self.l.gecc_microbench(self.h, which, iters, C.byref(r), C.byref(s), C.byref(t))
        if self._check(rc, "gecc_microbench"):
            raise ValueError(f"gecc_microbench rc={rc}")
        return dict(ops_per_clk_per_sm=r.value, seconds=s.value, total_ops=t.value)

    def bench_run(self, op: str, strategy: str, n: int, lanes: int = 0, workers: int = 0, seed: int = 1,
                  repeats: int = 5):
        """sm2b_bench_run (sm2batch.h:102-105); returns (status, report dict)."""

        class Report(C.Structure):
            _fields_ = [("lanes_used", C.c_uint64), ("wall_seconds", C.c_double), ("throughput", C.c_double),
                        ("ops", C.c_uint64 * 4), ("modeled_cost", C.c_uint64), ("equivalence_checked", C.c_int)]

        rep = Report()
        rc = self.l.sm2b_bench_run(self.h, op.encode(), strategy.encode(), C.c_size_t(n), C.c_size_t(lanes),
                                   C.c_uint32(workers), C.c_uint64(seed), C.c_uint32(repeats), C.byref(rep))
        self._check(rc, "sm2b_bench_run")
        return rc, dict(lanes_used=rep.lanes_used, wall_seconds=rep.wall_seconds, throughput=rep.throughput,
                        ops=dict(zip(("modmul", "modadd", "modsub", "modinv"), list(rep.ops))),
                        modeled_cost=rep.modeled_cost, equivalence_checked=rep.equivalence_checked)

    # -- batch layer (host column buffers)
    # ---- runtime moduli / user curves (gecc_*_rt): params from field_params_make(q)
    def field_op_rt(self, params, op: str, a: np.ndarray, b: np.ndarray | None = None):
        n = a.shape[1]
        _need_cols(a, 8, n, "field_op_rt a")
        if b is not None:
            _need_cols(b, 8, n, "field_op_rt b")
        out = np.zeros((8, n), np.uint32)
        rc = self.l.gecc_field_op_rt(self.h, params.ctypes.data, FIELD_OPS[op], C.c_size_t(n), _vp(a), _vp(b), _vp(out))
        if self._check(rc, "gecc_field_op_rt"):
            raise ValueError(f"gecc_field_op_rt rc={rc}")
        return out

    def batch_invert_rt(self, params, a: np.ndarray):
        n = a.shape[1]
        _need_cols(a, 8, n, "batch_invert_rt")
        out = np.zeros((8, n), np.uint32)
        rc = self.l.gecc_batch_invert_rt(self.h, params.ctypes.data, C.c_size_t(n), _vp(a), _vp(out))
        if self._check(rc, "gecc_batch_invert_rt"):
            raise ValueError(f"gecc_batch_invert_rt rc={rc}")
        return out

    def batch_padd_rt(self, params, a_mont: np.ndarray, P, T):
        n = P[0].shape[1]
        for X in (P, T):
            _need_cols(X[0], 8, n, "batch_padd_rt x")
            _need_cols(X[1], 8, n, "batch_padd_rt y")
            _need_mask(X[2], n, "batch_padd_rt infinity mask")
        ox, oy, oi = np.zeros((8, n), np.uint32), np.zeros((8, n), np.uint32), np.zeros(n, np.uint8)
        rc = self.l.gecc_batch_padd_rt(self.h, params.ctypes.data, a_mont.ctypes.data, C.c_size_t(n), _vp(P[0]), _vp(P[1]),
                                       _vp(P[2]), _vp(T[0]), _vp(T[1]), _vp(T[2]), _vp(ox), _vp(oy), _vp(oi))
        if self._check(rc, "gecc_batch_padd_rt"):
            raise ValueError(f"gecc_batch_padd_rt rc={rc}")
        return ox, oy, oi

    def batch_pdbl_rt(self, params, a_mont: np.ndarray, P):
        n = P[0].shape[1]
        _need_cols(P[0], 8, n, "batch_pdbl_rt x")
        _need_cols(P[1], 8, n, "batch_pdbl_rt y")
        _need_mask(P[2], n, "batch_pdbl_rt infinity mask")
        ox, oy, oi = np.zeros((8, n), np.uint32), np.zeros((8, n), np.uint32), np.zeros(n, np.uint8)
        rc = self.l.gecc_batch_pdbl_rt(self.h, params.ctypes.data, a_mont.ctypes.data, C.c_size_t(n), _vp(P[0]), _vp(P[1]),
                                       _vp(P[2]), _vp(ox), _vp(oy), _vp(oi))
        if self._check(rc, "gecc_batch_pdbl_rt"):
            raise ValueError(f"gecc_batch_pdbl_rt rc={rc}")
        return ox, oy, oi

    def batch_invert(self, field: int, a: np.ndarray):
        n = a.shape[1]
        _need_cols(a, self.limbs if field == 0 else 8, n, "batch_invert")
        out = np.zeros((self.limbs if field == 0 else 8, n), np.uint32)
        rc = self.l.gecc_batch_invert(self.h, field, C.c_size_t(n), _vp(a), _vp(out))
        if self._check(rc, "gecc_batch_invert"):
            raise ValueError(f"gecc_batch_invert rc={rc}")
        return out

    def _pts_out(self, n):
        return np.zeros((self.limbs, n), np.uint32), np.zeros((self.limbs, n), np.uint32), np.zeros(n, np.uint8)

    def _need_points(self, P, n, what):
        _need_cols(P[0], self.limbs, n, what + " x")
        _need_cols(P[1], self.limbs, n, what + " y")
        _need_mask(P[2], n, what + " infinity mask")

    def batch_padd(self, P, T):
        if P[0].shape != T[0].shape:
            raise ValueError("batch_padd: buffer sizes differ")  # batch_point.cpp:71-72
        n = P[0].shape[1]
        self._need_points(P, n, "batch_padd p")
        self._need_points(T, n, "batch_padd t")
        ox, oy, oi = self._pts_out(n)
        rc = self.l.gecc_batch_padd(self.h, C.c_size_t(n), _vp(P[0]), _vp(P[1]), _vp(P[2]),
                                    _vp(T[0]), _vp(T[1]), _vp(T[2]), _vp(ox), _vp(oy), _vp(oi))
        if self._check(rc, "gecc_batch_padd"):
            raise ValueError(f"gecc_batch_padd rc={rc}")
        return ox, oy, oi

    def batch_pdbl(self, P):
        n = P[0].shape[1]
        self._need_points(P, n, "batch_pdbl")
        ox, oy, oi = self._pts_out(n)
        rc = self.l.gecc_batch_pdbl(self.h, C.c_size_t(n), _vp(P[0]), _vp(P[1]), _vp(P[2]),
                                    _vp(ox), _vp(oy), _vp(oi))
        if self._check(rc, "gecc_batch_pdbl"):
            raise ValueError(f"gecc_batch_pdbl rc={rc}")
        return ox, oy, oi

    def batch_fpmul(self, scalars: np.ndarray, base: BaseTable | None = None):
        """scalars[i] * G, or scalars[i] * base for a precomputed table of another point."""
        n = scalars.shape[1]
        _need_cols(scalars, 8, n, "batch_fpmul scalars")
        ox, oy, oi = self._pts_out(n)
        if base is None:
            rc = self.l.gecc_batch_fpmul(self.h, C.c_size_t(n), _vp(scalars), _vp(ox), _vp(oy), _vp(oi))
        else:
            rc = self.l.gecc_batch_fpmul_base(self.h, base.h, C.c_size_t(n), _vp(scalars), _vp(ox), _vp(oy), _vp(oi))
        if self._check(rc, "gecc_batch_fpmul"):
            raise ValueError(f"gecc_batch_fpmul rc={rc}")
        return ox, oy, oi

    def base_table(self, x: np.ndarray, y: np.ndarray) -> BaseTable:
        return BaseTable(self, x, y)

    def batch_upmul(self, scalars: np.ndarray, P):
        n = scalars.shape[1]
        if P[0].shape[1] != n:
            raise ValueError("batch_upmul: scalar count mismatch")  # batch_point.cpp:239-240
        _need_cols(scalars, 8, n, "batch_upmul scalars")
        self._need_points(P, n, "batch_upmul")
        ox, oy, oi = self._pts_out(n)
        rc = self.l.gecc_batch_upmul(self.h, C.c_size_t(n), _vp(scalars), _vp(P[0]), _vp(P[1]),
                                     _vp(P[2]), _vp(ox), _vp(oy), _vp(oi))
        if self._check(rc, "gecc_batch_upmul"):
            raise ValueError(f"gecc_batch_upmul rc={rc}")
        return ox, oy, oi

    def msm(self, scalars: np.ndarray, P):
        n = scalars.shape[1]
        _need_cols(scalars, 8, n, "msm scalars")
        self._need_points(P, n, "msm")
        ox, oy, oi = self._pts_out(1)
        rc = self.l.gecc_msm(self.h, C.c_size_t(n), _vp(scalars), _vp(P[0]), _vp(P[1]), _vp(P[2]),
                             _vp(ox), _vp(oy), _vp(oi))
        if self._check(rc, "gecc_msm"):
            raise ValueError(f"gecc_msm rc={rc}")
        return ox, oy, oi

    # -- protocol layer (byte records, sm2batch.h:61-82)
    def keygen(self, seed: int, count: int, lane_base: int = 0):
        sec = (C.c_uint8 * max(1, 32 * count))()
        pub = (C.c_uint8 * max(1, 65 * count))()
        rc = self.l.gecc_keygen(self.h, C.c_uint64(seed), C.c_uint64(lane_base), C.c_size_t(count),
                                sec, pub)
        self._check(rc, "gecc_keygen")
        return rc, bytes(sec)[:32 * count], bytes(pub)[:65 * count]

    def sign(self, digests: bytes, secrets: bytes, nonce_seed: int, lane_base: int = 0,
             want_status: bool = True):
        count = len(digests) // 32
        _need_bytes(digests, 32 * count, "sign digests")
        _need_bytes(secrets, 32 * count, "sign secrets")
        sig = (C.c_uint8 * max(1, 64 * count))()
        st = (C.c_int32 * max(1, count))() if want_status else None
        rc = self.l.gecc_sign(self.h, C.c_size_t(count), _vp(digests), _vp(secrets),
                              C.c_uint64(nonce_seed), C.c_uint64(lane_base), sig, st)
        self._check(rc, "gecc_sign")
        return rc, bytes(sig)[:64 * count], (list(st)[:count] if st is not None else None)

    def sign_nonces(self, digests: bytes, secrets: bytes, nonces: bytes, want_status: bool = True):
        """One signing attempt with caller-supplied nonces (gecc_sign_nonces); status 5 = replace."""
        count = len(digests) // 32
        _need_bytes(digests, 32 * count, "sign_nonces digests")
        _need_bytes(secrets, 32 * count, "sign_nonces secrets")
        _need_bytes(nonces, 32 * count, "sign_nonces nonces")
        sig = (C.c_uint8 * max(1, 64 * count))()
        st = (C.c_int32 * max(1, count))() if want_status else None
        rc = self.l.gecc_sign_nonces(self.h, C.c_size_t(count), _vp(digests), _vp(secrets), _vp(nonces), sig, st)
        self._check(rc, "gecc_sign_nonces")
        return rc, bytes(sig)[:64 * count], (list(st)[:count] if st is not None else None)

    def verify(self, digests: bytes, publics: bytes, sigs: bytes):
        count = len(digests) // 32
        _need_bytes(digests, 32 * count, "verify digests")
        _need_bytes(publics, 65 * count, "verify publics")
        _need_bytes(sigs, 64 * count, "verify signatures")
        res = (C.c_uint8 * max(1, count))()
        rc = self.l.sm2b_verify(self.h, C.c_size_t(count), _vp(digests), _vp(publics), _vp(sigs), res)
        self._check(rc, "sm2b_verify")
        return rc, bytes(res)[:count]

    def ecdh(self, secrets: bytes, peers: bytes, want_status: bool = True):
        count = len(secrets) // 32
        _need_bytes(secrets, 32 * count, "ecdh secrets")
        _need_bytes(peers, 65 * count, "ecdh peers")
        sh = (C.c_uint8 * max(1, 32 * count))()
        st = (C.c_int32 * max(1, count))() if want_status else None
        rc = self.l.sm2b_ecdh(self.h, C.c_size_t(count), _vp(secrets), _vp(peers), sh, st)
        self._check(rc, "sm2b_ecdh")
        return rc, bytes(sh)[:32 * count], (list(st)[:count] if st is not None else None)
