#!/usr/bin/env python
"""bench.py -- headline benchmark: secp256k1 ECDSA verify, batch 2^20 per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload verify|sign|padd] [--log2n 20]

One JSON line on stdout (rank 0).  A "step" is one pass of the hot path over one
batch of synthetic records (BASELINE.json configs[1]: 2^20 signatures per GPU).

  value     whole-job throughput with the records already resident in HBM
            (CUDA events on the stream the kernel is launched on, max over ranks)
  e2e       the same metric through the reference-facing C ABI (sm2b_verify on a
            secp256k1 context): pinned HOST buffers in, host results out, the
            host<->device copies inside the timed region
  roofline  integer-multiply (IMAD) pipe: executed field multiplications x
            multiply-issue slots each, against the pipe peak measured live by
            the library's own microbenchmark in the same process
  cpu_baseline  the reference's CPU path on this box's host cores on a bounded
            sample of the same records (oracle/_ref, else the C port)

N > 1: launched by torchrun, one rank per GPU; lanes are sharded by range with
the global lane index as nonce stream, no data-path collective (scaling: weak).
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SECP = 1          # curve id of the oracle / reference shim; --curve sm2 switches it to 0 (the reference's own curve)
METRIC = {"verify": "ecdsa_verify_throughput", "sign": "ecdsa_sign_throughput",
          "padd": "batch_padd_throughput", "msm": "msm_time"}
UNIT = {"verify": "verifications/s", "sign": "signatures/s", "padd": "point additions/s",
        "msm": "ms per MSM"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="verify", choices=["verify", "sign", "padd", "msm"])
    ap.add_argument("--log2n", type=int, default=20)
    ap.add_argument("--curve", default="secp256k1", choices=["secp256k1", "sm2", "bls12_381", "bls12_377"],
                    help="sm2 = the reference's own curve; bls12_381 / bls12_377 (12-limb coordinates) are served by --workload msm only")
    ap.add_argument("--cpu-sample-log2", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="headline leg only (default: the verify headline also carries sign / MSM / padd legs in `extra`)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML polled every 5 ms from a
    thread (short timed regions still get samples), `nvidia-smi -lms` (the profiling recipe's
    line) when the NVML binding is missing."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.rows, self.proc, self.nv = [], None, None
        self.sm, self.mx, self.reasons, self.stop_flag = [], None, set(), False
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.nv = nv
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _poll(self):
        nv = self.nv
        get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        while not self.stop_flag:
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = int(get(self.h))
                for nm, b in bits.items():
                    if r & b:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.nv is not None:
            self.stop_flag = True
            self.t.join(timeout=1)
            return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.mx,
                    "samples": len(self.sm), "reasons": sorted(self.reasons), "source": "nvml, 5 ms period"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(self.NAMES, r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons), "source": "nvidia-smi -lms 100"}


# ----------------------------------------------------------------------------- CPU arm
def cpu_verify_runner():
    """Returns (kind, cores, fn(dig, pub, sig) -> results) for the CPU reference path."""
    from oracle import refshim as R
    if R.available():
        cores = os.cpu_count() or 1
        return "reference", cores, lambda d, p, s: R.ecdsa_verify(SECP, d, p, s, workers=0)[1]
    from oracle import coracle as O
    return "port", 1, lambda d, p, s: O.ecdsa_verify(SECP, d, p, s)[1]


def cpu_sign_runner():
    from oracle import refshim as R
    if R.available():
        cores = os.cpu_count() or 1
        return "reference", cores, lambda d, s, seed: R.ecdsa_sign(SECP, d, s, seed, workers=0)[1]
    from oracle import coracle as O
    return "port", 1, lambda d, s, seed: O.ecdsa_sign(SECP, d, s, seed)[1]


def make_records_cpu(n, seed=1):
    """Synthetic keys/digests/signatures for the reference arm, made by the CPU path itself."""
    from oracle import refshim as R
    from oracle import coracle as O
    import numpy as np
    src = R if R.available() else O
    kw = {"workers": 0} if R.available() else {}
    rc, sec, pub = src.keygen(SECP, seed, n, **kw)
    dig = np.random.RandomState(seed).bytes(32 * n)
    rc, sig, st = src.ecdsa_sign(SECP, dig, sec, seed + 1, **kw)
    return dig, sec, pub, sig


def set_curve(args):
    global SECP
    SECP = 0 if args.curve == "sm2" else 1


def reference_arm_points(args, wl):
    """padd: the reference's batch_padd (all host threads) on 2^16 pairs per step.  msm: the
    reference has none -- its serial scalar multiplication over 2^11 terms per step, scaled to
    the 2^log2n terms of the workload (what a caller of the reference would have to run)."""
    import numpy as np
    from oracle import refshim as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref is not built"}), flush=True)
        return
    cores = os.cpu_count()
    m = 1 << (args.cpu_sample_log2 or (16 if wl == "padd" else 11))
    rs = np.random.RandomState(99)
    k1 = rs.randint(0, 2**32, size=(8, m), dtype=np.uint64).astype(np.uint32)
    k2 = rs.randint(0, 2**32, size=(8, m), dtype=np.uint64).astype(np.uint32)
    P = R.batch_fpmul(SECP, k1, workers=0)
    if wl == "padd":
        T = R.batch_fpmul(SECP, k2, workers=0)
        step = lambda: R.batch_padd(SECP, P, T, lanes=0, workers=0)
        used = cores
    else:
        step = lambda: R.pmul_serial(SECP, k2, P)
        used = 1
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    n = 1 << args.log2n
    value = m / dt if wl == "padd" else dt * (n / m) * 1e3
    sample = (f"2^{m.bit_length() - 1} pairs per step, reference batch_padd" if wl == "padd" else
              f"reference pmul_serial over 2^{m.bit_length() - 1} terms per step, scaled by {n // m} to 2^{args.log2n} terms (the reference has no MSM)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC[wl], "value": value, "unit": UNIT[wl], "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": wl != "msm",
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 limbs (256-bit modular integer)", "data": "synthetic",
        "config": {"workload": f"{args.curve} {'batched affine point addition' if wl == 'padd' else 'Pippenger MSM'}, 2^{args.log2n} per GPU",
                   "curve": args.curve, "cpu_sample_per_step": m},
        "cpu_baseline": {"value": value, "unit": UNIT[wl], "cores": used, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT[wl], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0}), flush=True)


def run_reference_arm(args, rank):
    set_curve(args)
    if rank != 0:
        return
    wl = args.workload
    if wl in ("padd", "msm") and args.curve in ("secp256k1", "sm2"):
        reference_arm_points(args, wl)
        return
    if wl not in ("verify", "sign"):
        print(json.dumps({"impl": "reference", "unavailable": f"the reference has no {args.curve} {wl}"}), flush=True)
        return
    # 2^16 lanes per step: the reference's throughput is flat beyond 2^12 but a 2^13 sample under-reports
    # it by ~28 % (BENCH_r01: 12.9 k/s at 2^13 against 17.9 k/s at 2^16 on the same box)
    log2 = args.cpu_sample_log2 or 16
    n = 1 << log2
    dig, sec, pub, sig = make_records_cpu(n)
    if wl == "verify":
        kind, cores, fn = cpu_verify_runner()
        step = lambda: fn(dig, pub, sig)
    else:
        kind, cores, fn = cpu_sign_runner()
        step = lambda: fn(dig, sec, 7)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = step()
    dt = time.perf_counter() - t0
    if wl == "verify":
        assert out == b"\x01" * n
    value = n * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC[wl], "value": value, "unit": UNIT[wl],
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 limbs (256-bit modular integer)", "data": "synthetic",
        "config": {"workload": f"{args.curve} ECDSA {wl}, batch 2^{args.log2n} per GPU",
                   "curve": args.curve, "cpu_sample_lanes_per_step": n},
        "cpu_baseline": {"value": value, "unit": UNIT[wl], "cores": cores, "kind": kind,
                         "sample": f"2^{log2} lanes per step of the same synthetic recipe; "
                                   "reference batch kernels (batch_fpmul/upmul/padd/invert) driven by "
                                   + ("the protocol glue that is checked equal to the reference's sm2b_sign / sm2b_verify"
                                      if args.curve == "sm2" else "the restated secp256k1 protocol glue")},
        "e2e": {"value": value, "unit": UNIT[wl], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
# Executed field products per lane of OUR kernels: counted by running the product's own
# lane code on the host with instrumented multiply / square / safegcd
# (tools/count_ops.py -> tools/op_counts.json; method in DESIGN.md "work per lane").
# Roofline unit = one IMAD.WIDE (32 x 32 -> 64 multiply-add), the instruction whose issue rate
# (32 per clk per SM) bounds the path.  ONLY IMAD.WIDE is counted per product -- the 32-bit IMAD
# / IMAD.HI a reduction also issues are overhead, not work -- so the figure can be checked
# against the ncu opcode mix (profiles/*_opmix.csv: IMAD.WIDE warp instructions x active lanes).
SLOTS = {
    "mul_special": 64 + 8,             # 8 x 8 product + the 8 wide multiplies of the pseudo-Mersenne fold
    "sqr_special": 36 + 8,
    "mul_generic": 64 + 64,            # product + word-serial Montgomery rows (m_i * q)
    "sqr_generic": 36 + 64,
    "safegcd_special": 20 * (36 + 54),  # 20 rounds of two 2x2 matrix updates on 9 limbs
    "safegcd_generic": 20 * (36 + 54),
}
IO_BYTES = {"verify": 162, "sign": 132, "padd": 194, "msm": 96}   # algorithmic bytes per unit
KERNEL = {"verify": "k_verify_gtab", "sign": "k_sign", "padd": "k_batch_padd", "msm": "k_msm_*"}


def msm_products_per_point(kind, log2n=20, windows=17, bucket_bits=15):
    """Executed field products per input point of the batch-affine MSM: `windows` x (1 - 1/32)
    tree joins, each 5 mul + 1 sqr (denominator product, two unwind products, lambda, lambda^2, y)
    plus its share of the block scan (1.2 per join on average); then the three marginal sums:
    3 x 1.5 mixed Jacobian additions (8M + 3S) per BUCKET, windows x 2^bucket_bits buckets."""
    joins = windows * (1 - 1 / 32)
    madds = 3 * 1.5 * windows * 2**bucket_bits / 2**log2n
    return {f"mul_{kind}": joins * (5 + 1.2) + madds * 8, f"sqr_{kind}": joins * 1 + madds * 3}


def work_per_lane(workload, curve="secp256k1", log2n=20, msm_shape=None):
    with open(os.path.join(ROOT, "tools", "op_counts.json")) as f:
        counts = json.load(f)[curve]
    if workload == "padd":   # ALGORITHMIC work of one affine addition under Montgomery's trick:
        c = {"mul_special": 5, "sqr_special": 1}   # 6 products per pair; the shared inversion is not counted
    elif workload == "msm":
        c = msm_products_per_point("special", log2n, *(msm_shape or (17, 15)))
    else:
        c = counts[workload]
    table = dict(SLOTS)
    if curve == "sm2":   # SM2 p: the reduction is additions and subtractions only (field.cpp:88-128)
        table.update(mul_special=64, sqr_special=36)
    slots = sum(table[k] * v for k, v in c.items())
    products = sum(v for k, v in c.items() if not k.startswith("safegcd"))
    return c, slots, products


class GpuArm:
    """Synthetic records + device buffers of one rank, and the timed legs over them."""

    def __init__(self, args, rank, local_rank, world):
        import numpy as np
        import torch
        import torch.distributed as dist
        import paper_2501_03245_b200 as gecc
        self.np, self.torch, self.dist, self.gecc = np, torch, dist, gecc
        self.args, self.rank, self.local_rank, self.world = args, rank, local_rank, world
        if not torch.cuda.is_available():
            raise SystemExit("bench.py: no CUDA device; the product has no CPU path "
                             "(use --impl reference for the CPU arm)")
        torch.cuda.set_device(local_rank)
        if world > 1 or (os.environ.get("GECC_BENCH_FORCE_EXCHANGE") == "1" and "RANK" in os.environ):
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        self.ctx = gecc.Context(gecc.SM2 if args.curve == "sm2" else gecc.SECP256K1, local_rank)
        self.l = gecc.lib()
        self.stream = torch.cuda.Stream()          # all timed work and its events share this stream
        torch.cuda.set_stream(self.stream)
        self.ctx.set_stream(self.stream.cuda_stream)
        peak = self.ctx.microbench(1, 3000)        # dependent IMAD.WIDE chain, 8 warps per scheduler
        self.peak = peak
        self.peak_mad_per_s = peak["total_ops"] / peak["seconds"]
        self.records = {}
        self.points = {}
        self.comm_ready = False

    # ---- plumbing
    def vp(self, t):
        return C.c_void_p(t.data_ptr())

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()
            self.torch.cuda.synchronize()

    def max_over_ranks(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def pin(self, a):
        return self.torch.from_numpy(a).pin_memory()

    # ---- synthetic inputs, generated on the GPU by our own keygen / sign / fpmul (not timed)
    def ensure_records(self, n):
        if n in self.records:
            return self.records[n]
        np, torch, l, ctx, vp = self.np, self.torch, self.l, self.ctx, self.vp
        lane_base = self.rank * n
        h_sec, h_pub = np.empty(32 * n, np.uint8), np.empty(65 * n, np.uint8)
        rc = l.gecc_keygen(ctx.h, C.c_uint64(1), C.c_uint64(lane_base), C.c_size_t(n),
                           C.c_void_p(h_sec.ctypes.data), C.c_void_p(h_pub.ctypes.data))
        assert rc == 0, l.gecc_last_error(ctx.h)
        h_dig = np.frombuffer(np.random.RandomState(1234 + self.rank).bytes(32 * n), np.uint8).copy()
        d_dig, d_sec, d_pub = (torch.from_numpy(a).cuda() for a in (h_dig, h_sec, h_pub))
        d_sig = torch.empty(64 * n, dtype=torch.uint8, device="cuda")
        d_res = torch.empty(n, dtype=torch.uint8, device="cuda")
        d_st = torch.empty(n, dtype=torch.int32, device="cuda")
        rc = l.gecc_sign_dev(ctx.h, C.c_size_t(n), vp(d_dig), vp(d_sec), C.c_uint64(7),
                             C.c_uint64(lane_base), vp(d_sig), vp(d_st))
        assert rc == 0
        torch.cuda.synchronize()
        assert int(d_st.abs().sum()) == 0
        h_sig = d_sig.cpu().numpy()
        # equivalence gate before timing (bench.cpp:253-256): spot lanes vs the oracle
        from oracle import coracle as O
        rs = np.random.RandomState(99)
        idx = [int(i) for i in rs.choice(n, 24, replace=False)]
        pick = lambda a, w: b"".join(a[w * i:w * i + w].tobytes() for i in idx)
        for i in idx[:8]:
            want = O.ecdsa_sign(SECP, h_dig[32 * i:32 * i + 32].tobytes(), h_sec[32 * i:32 * i + 32].tobytes(),
                                7, lane_base=lane_base + i)[1]
            assert want == h_sig[64 * i:64 * i + 64].tobytes(), "sign parity gate failed"
        bad = bytearray(pick(h_sig, 64))
        bad[64 * 3 + 9] ^= 4
        want = O.ecdsa_verify(SECP, pick(h_dig, 32), pick(h_pub, 65), bytes(bad))[1]
        got = ctx.verify(pick(h_dig, 32), pick(h_pub, 65), bytes(bad))[1]
        assert want == got and sum(want) == 23, "verify parity gate failed"
        r = dict(n=n, lane_base=lane_base, h_dig=h_dig, h_sec=h_sec, h_pub=h_pub, h_sig=h_sig, d_dig=d_dig,
                 d_sec=d_sec, d_pub=d_pub, d_sig=d_sig, d_res=d_res, d_st=d_st)
        self.records[n] = r
        return r

    def ensure_points(self, n):
        if n in self.points:
            return self.points[n]
        np, torch, l, ctx, vp = self.np, self.torch, self.l, self.ctx, self.vp
        rs = np.random.RandomState(99 + self.rank)
        k1 = torch.from_numpy(rs.randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32)).cuda()
        k2 = torch.from_numpy(rs.randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32)).cuda()
        col = lambda m=n: torch.empty((8, m), dtype=torch.int32, device="cuda")
        u8 = lambda m: torch.empty(m, dtype=torch.uint8, device="cuda")
        P = (col(), col(), u8(n)); T = (col(), col(), u8(n)); S = (col(), col(), u8(n))
        assert l.gecc_batch_fpmul_dev(ctx.h, C.c_size_t(n), vp(k1), vp(P[0]), vp(P[1]), vp(P[2])) == 0
        assert l.gecc_batch_fpmul_dev(ctx.h, C.c_size_t(n), vp(k2), vp(T[0]), vp(T[1]), vp(T[2])) == 0
        torch.cuda.synchronize()
        M = (col(1), col(1), u8(1))
        p = dict(n=n, k1=k1, k2=k2, P=P, T=T, S=S, M=M)
        self.points[n] = p
        return p

    def ensure_comm(self):
        """MSM exchange communicator in the library (ncclCommInitRank); torch.distributed only
        carries the 128-byte id from rank 0."""
        if self.comm_ready:
            return
        uid = [self.gecc.comm_unique_id() if self.rank == 0 else None]
        if self.world > 1:
            self.dist.broadcast_object_list(uid, src=0)
        self.ctx.comm_init_rank(self.world, self.rank, uid[0])
        self.comm_ready = True

    # ---- one leg: device-resident value, e2e through the host API, roofline, CPU baseline
    def run(self, wl, log2n, with_cpu=True):
        np, torch, l, ctx, vp, args = self.np, self.torch, self.l, self.ctx, self.vp, self.args
        n = 1 << log2n
        world, rank = self.world, self.rank
        stream = self.stream
        msm_exchange = wl == "msm" and (world > 1 or os.environ.get("GECC_BENCH_FORCE_EXCHANGE") == "1")
        if wl in ("verify", "sign"):
            r = self.ensure_records(n)
            lane_base = r["lane_base"]
        else:
            p = self.ensure_points(n)
            P, T, S, M = p["P"], p["T"], p["S"], p["M"]
            if msm_exchange:
                self.ensure_comm()

        def step_dev():
            if wl == "verify":
                return l.gecc_verify_dev(ctx.h, C.c_size_t(n), vp(r["d_dig"]), vp(r["d_pub"]), vp(r["d_sig"]), vp(r["d_res"]))
            if wl == "sign":
                return l.gecc_sign_dev(ctx.h, C.c_size_t(n), vp(r["d_dig"]), vp(r["d_sec"]), C.c_uint64(7),
                                       C.c_uint64(lane_base), vp(r["d_sig"]), vp(r["d_st"]))
            if wl == "msm":   # sum_i k2_i * P_i, one point out
                rc = l.gecc_msm_dev(ctx.h, C.c_size_t(n), vp(p["k2"]), vp(P[0]), vp(P[1]), vp(P[2]),
                                    vp(M[0]), vp(M[1]), vp(M[2]))
                if not msm_exchange or rc != 0:
                    return rc
                # sharded MSM: every rank summed its own point range; the library
                # all-gathers the partial sums over NCCL and adds them locally, in C++
                return l.gecc_msm_combine_dev(ctx.h, vp(M[0]), vp(M[1]), vp(M[2]))
            return l.gecc_batch_padd_dev(ctx.h, C.c_size_t(n), vp(P[0]), vp(P[1]), vp(P[2]), vp(T[0]),
                                         vp(T[1]), vp(T[2]), vp(S[0]), vp(S[1]), vp(S[2]))

        # ---- value: device-resident
        for _ in range(args.warmup):
            assert step_dev() == 0
        self.barrier()
        sampler = ClockSampler(self.local_rank)
        launches0 = ctx.launches
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            assert step_dev() == 0
        ev1.record(stream)
        self.barrier()
        launches = ctx.launches - launches0
        dev_s = self.max_over_ranks(ev0.elapsed_time(ev1) * 1e-3)
        clocks = sampler.stop()
        if wl == "verify":
            assert int(r["d_res"].sum()) == n, "timed verify produced rejects"
        per_launch_s = dev_s / args.steps
        value = world * n * args.steps / dev_s
        if wl == "msm":   # time-like metric: ms per 2^log2n-point MSM (per GPU; ranks run their own range)
            value = per_launch_s * 1e3

        # ---- e2e: reference-facing C ABI, pinned host buffers, copies inside the timed region
        pin = self.pin
        if wl in ("verify", "sign"):
            p_dig, p_pub, p_sig, p_sec = pin(r["h_dig"]), pin(r["h_pub"]), pin(r["h_sig"].copy()), pin(r["h_sec"])
            p_res = torch.empty(n, dtype=torch.uint8).pin_memory()
            p_out = torch.empty(64 * n, dtype=torch.uint8).pin_memory()
            p_st = torch.empty(n, dtype=torch.int32).pin_memory()
            if wl == "verify":
                call = lambda: l.sm2b_verify(ctx.h, C.c_size_t(n), vp(p_dig), vp(p_pub), vp(p_sig), vp(p_res))
                h2d, d2h, api = 161 * n, n, "sm2b_verify"
            else:
                call = lambda: l.gecc_sign(ctx.h, C.c_size_t(n), vp(p_dig), vp(p_sec), C.c_uint64(7),
                                           C.c_uint64(lane_base), vp(p_out), vp(p_st))
                h2d, d2h, api = 64 * n, 68 * n, "gecc_sign"
        else:
            h = lambda t, i: pin(np.ascontiguousarray(t.cpu().numpy().view(np.uint32 if i < 2 else np.uint8)))
            hP = tuple(h(t, i) for i, t in enumerate(P))
            hT = tuple(h(t, i) for i, t in enumerate(T))
            hk = pin(p["k2"].cpu().numpy())
            m_out = n if wl == "padd" else 1
            hO = (torch.empty((8, m_out), dtype=torch.int32).pin_memory(), torch.empty((8, m_out), dtype=torch.int32).pin_memory(),
                  torch.empty(m_out, dtype=torch.uint8).pin_memory())
            if wl == "padd":
                call = lambda: l.gecc_batch_padd(ctx.h, C.c_size_t(n), vp(hP[0]), vp(hP[1]), vp(hP[2]), vp(hT[0]), vp(hT[1]),
                                                 vp(hT[2]), vp(hO[0]), vp(hO[1]), vp(hO[2]))
                h2d, d2h, api = 130 * n, 65 * n, "gecc_batch_padd"
            else:
                call = lambda: l.gecc_msm(ctx.h, C.c_size_t(n), vp(hk), vp(hP[0]), vp(hP[1]), vp(hP[2]),
                                          vp(hO[0]), vp(hO[1]), vp(hO[2]))
                h2d, d2h, api = 97 * n, 65, "gecc_msm"
        for _ in range(max(1, args.warmup // 2)):
            assert call() == 0
        self.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            assert call() == 0  # synchronous: returns after the D2H copy completed
        torch.cuda.synchronize()
        e2e_s = self.max_over_ranks(time.perf_counter() - t0)
        if wl == "verify":
            assert int(p_res.sum()) == n
        elif wl == "sign":   # deterministic nonces: the pipelined host path must reproduce the device path's bytes
            assert bytes(p_out.numpy()[:4096]) == r["h_sig"][:4096].tobytes() and int(p_st.abs().sum()) == 0
            assert bytes(p_out.numpy()[-4096:]) == r["h_sig"][-4096:].tobytes()
        e2e = {"value": (e2e_s / args.steps * 1e3) if wl == "msm" else world * n * args.steps / e2e_s, "unit": UNIT[wl],
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s / args.steps * 1e3,
               "api": api, "host_buffers": "pinned"}

        # ---- roofline of the dominant kernel
        counts, slots_per_lane, products_per_lane = work_per_lane(wl, args.curve, log2n)
        achieved = n * slots_per_lane / per_launch_s
        io_bytes = IO_BYTES[wl] * n
        hbm_peak = _measured_peaks().get("hbm_gbs")
        roofline = {
            "bound": "imad", "kernel": KERNEL[wl],
            "achieved": achieved / 1e12, "peak": self.peak_mad_per_s / 1e12, "unit": "T IMAD.WIDE/s",
            "frac": achieved / self.peak_mad_per_s,
            "peak_source": "measured live: gecc_microbench(dependent IMAD.WIDE.U32), "
                           f"{self.peak['ops_per_clk_per_sm']:.1f} per clk per SM (MEASURED_PEAKS.json has no integer peak)",
            "work_per_unit": {"executed": counts, "imad_wide": slots_per_lane, "imad_wide_per_op": SLOTS,
                              "source": "tools/op_counts.json (host-sim counted)" if wl in ("verify", "sign")
                              else "algorithmic count (DESIGN.md section 4)"},
            "modmul_per_s": n * products_per_lane / per_launch_s,
            "hbm": {"algorithmic_bytes_per_launch": io_bytes, "achieved_gbs": io_bytes / per_launch_s / 1e9,
                    "peak_gbs": hbm_peak, "frac": (io_bytes / per_launch_s / 1e9 / hbm_peak) if hbm_peak else None,
                    "note": "records only" + ("; near the compute / HBM ridge" if wl == "padd" else "; not the bound")},
            "traffic": _ncu_traffic(wl, log2n) if args.curve == "secp256k1" else None,
        }

        # ---- CPU baseline on this box's host cores (rank 0, N = 1 only): the compiled reference on a
        # bounded sample of the SAME inputs, outputs compared with the GPU's
        cpu = None
        if with_cpu and rank == 0 and world == 1 and not args.no_cpu_baseline:
            cpu = self.cpu_baseline(wl, n, log2n, locals())
        return {"metric": METRIC[wl], "value": value, "unit": UNIT[wl], "ms_per_step": per_launch_s * 1e3,
                "higher_is_better": wl != "msm", "lanes_per_gpu": n, "clocks": clocks, "e2e": e2e,
                "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu}

    def cpu_baseline(self, wl, n, log2n, env):
        np, args = self.np, self.args
        if wl in ("verify", "sign"):
            r = env["r"]
            log2 = args.cpu_sample_log2 or (16 if wl == "verify" else 17)
            m = min(n, 1 << log2)
            if wl == "verify":
                kind, cores, fn = cpu_verify_runner()
                if kind == "port":
                    m = min(m, 1 << 12)
                t0 = time.perf_counter()
                out = fn(r["h_dig"][:32 * m].tobytes(), r["h_pub"][:65 * m].tobytes(), r["h_sig"][:64 * m].tobytes())
                dt = time.perf_counter() - t0
                assert out == b"\x01" * m, "CPU reference rejected GPU-made signatures"
            else:
                kind, cores, fn = cpu_sign_runner()
                if kind == "port":
                    m = min(m, 1 << 13)
                t0 = time.perf_counter()
                out = fn(r["h_dig"][:32 * m].tobytes(), r["h_sec"][:32 * m].tobytes(), 7)
                dt = time.perf_counter() - t0
                assert out == r["h_sig"][:64 * m].tobytes(), "CPU reference signatures differ from the GPU's"
            return {"value": m / dt, "unit": UNIT[wl], "cores": cores, "kind": kind,
                    "sample": f"first {m} lanes of the timed batch, one call, outputs compared with the GPU's",
                    "seconds": dt}
        from oracle import refshim as R
        if not R.available():
            return None
        P, T, hO, k2 = env["P"], env["T"], env["hO"], env["p"]["k2"]
        m = min(n, 1 << (16 if wl == "padd" else 11))
        cut = lambda t, w: np.ascontiguousarray(t.cpu().numpy().view(w)[..., :m])
        cP = (cut(P[0], np.uint32), cut(P[1], np.uint32), cut(P[2], np.uint8))
        if wl == "padd":   # the reference's batch_padd on all host threads, up to 2^16 pairs, median of 5
            cT = (cut(T[0], np.uint32), cut(T[1], np.uint32), cut(T[2], np.uint8))
            dt = R.batch_padd_timed(SECP, cP, cT, lanes=0, workers=0, repeats=5)
            want = R.batch_padd(SECP, cP, cT, lanes=0, workers=0)
            got = tuple(np.ascontiguousarray(t.numpy().view(w)[..., :m]) for t, w in zip(hO, (np.uint32, np.uint32, np.uint8)))
            assert all((a == b).all() for a, b in zip(want, got)), "CPU reference batch_padd differs from the GPU's"
            return {"value": m / dt, "unit": UNIT[wl], "cores": os.cpu_count(), "kind": "reference",
                    "sample": f"first {m} pairs of the timed batch, median of 5, ALL outputs compared with the GPU's",
                    "seconds": dt}
        # the reference has no MSM: its serial scalar multiplication (pmul_serial) summed, 2^11 terms
        ck = np.ascontiguousarray(k2.cpu().numpy()[..., :m])
        t0 = time.perf_counter()
        R.pmul_serial(SECP, ck, cP)
        dt = time.perf_counter() - t0
        return {"value": dt * (n / m) * 1e3, "unit": UNIT[wl], "cores": 1, "kind": "reference",
                "sample": f"reference pmul_serial over the first {m} terms ({dt:.2f} s), scaled by {n // m} to 2^{log2n} "
                          "terms; the reference has no MSM, this is the definition it would run",
                "seconds": dt}

    def close(self):
        self.ctx.close()
        if self.dist.is_initialized():
            self.dist.destroy_process_group()


WORKLOAD_TEXT = {"verify": "{c} ECDSA verify, batch 2^{k} per GPU", "sign": "{c} ECDSA sign, batch 2^{k} per GPU",
                 "padd": "{c} batched affine point addition, 2^{k} pairs per GPU",
                 "msm": "{c} Pippenger MSM, 2^{k} points per GPU (batch-affine buckets)"}
# the other legs of BASELINE.json's metric ("ECDSA sign & verify ops/s ...; MSM 2^20 ms") and config 1
EXTRA_LEGS = [("sign_2^20", "sign", 20), ("msm_2^20", "msm", 20), ("padd_2^16", "padd", 16), ("padd_2^20", "padd", 20)]


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    set_curve(args)
    if args.curve.startswith("bls"):
        if args.workload != "msm":
            raise SystemExit("bench.py: the BLS curves serve --workload msm only")
        bench_msm_bls(args, rank, local_rank, world)
        return
    arm = GpuArm(args, rank, local_rank, world)
    wl = args.workload
    leg = arm.run(wl, args.log2n)
    extra = None
    if wl == "verify" and args.log2n == 20 and not args.no_extra:
        extra = {}
        for name, w, k in EXTRA_LEGS:
            e = arm.run(w, k)
            e["config"] = {"workload": WORKLOAD_TEXT[w].format(c=args.curve, k=k)}
            extra[name] = e
    if rank == 0:
        line = {
            "metric": leg["metric"], "value": leg["value"], "unit": leg["unit"], "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": leg["ms_per_step"],
            "higher_is_better": leg["higher_is_better"], "scaling": "weak", "vs_baseline": None,
            "dtype": "u32 limbs (256-bit modular integer)", "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT[wl].format(c=args.curve, k=args.log2n),
                       "curve": args.curve, "lanes_per_gpu": 1 << args.log2n,
                       "sharding": (f"point ranges x{world}, one ncclAllGather of the partial sums + {world - 1} local additions (in the library)"
                                    if wl == "msm" and world > 1 else f"lane ranges x{world}, no collective"),
                       "l2": "inputs larger than L2 (records 161 B/lane x 2^20 = 169 MB > 126 MB)"
                       if wl == "verify" and args.log2n >= 20 else "no L2 flush; kernel is IMAD-bound, records read once",
                       "parity": "secp256k1 ECDSA: pinned to reference kernels + restated protocol glue + Python ints; "
                                 "MSM: definition only (the reference has none)"},
            "clocks": leg["clocks"], "e2e": leg["e2e"], "gpu_launches": leg["gpu_launches"],
            "roofline": leg["roofline"], "cpu_baseline": leg["cpu_baseline"],
        }
        if extra is not None:
            line["extra"] = extra
        print(json.dumps(line), flush=True)
    arm.close()


def bench_msm_bls(args, rank, local_rank, world):
    """BLS12-381 / BLS12-377 G1 MSM (12-limb coordinates, 255 / 253-bit group order), device-resident.  Points are
    i * G for i = 1 .. n, built on the GPU by doubling-and-adding whole arrays (batch_padd /
    batch_pdbl); the gate before timing checks sum_i k_i (i G) = (sum_i k_i i mod r) G against
    Python integers."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2501_03245_b200 as gecc
    from oracle import pyec as E   # equivalence gate only

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    B = E.CURVES[args.curve]
    n = 1 << args.log2n
    ctx = gecc.Context(gecc.BLS12_381 if args.curve == "bls12_381" else gecc.BLS12_377, local_rank)
    l = gecc.lib()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    vp = lambda t: C.c_void_p(t.data_ptr())
    R12 = 1 << 384
    g = (gecc.cols_from_ints([B.gx * R12 % B.p], 12), gecc.cols_from_ints([B.gy * R12 % B.p], 12), np.zeros(1, np.uint8))
    # [1..2^k - 1] G  ->  [1..2^(k+1) - 1] G  =  old, 2^k G, old + 2^k G
    px, py = torch.from_numpy(g[0].copy()).cuda().view(torch.int32), torch.from_numpy(g[1].copy()).cuda().view(torch.int32)
    base = (px.clone(), py.clone())
    zero = lambda m: torch.zeros(m, dtype=torch.uint8, device="cuda")
    col = lambda m: torch.empty((12, m), dtype=torch.int32, device="cuda")
    for _ in range(args.log2n - 1):
        m = px.shape[1]
        bx, by = base[0].expand(12, m).contiguous(), base[1].expand(12, m).contiguous()
        ox, oy, oi = col(m), col(m), zero(m)
        assert l.gecc_batch_padd_dev(ctx.h, C.c_size_t(m), vp(px), vp(py), None, vp(bx), vp(by), None,
                                     vp(ox), vp(oy), vp(oi)) == 0
        px, py = torch.cat([px, base[0], ox], 1).contiguous(), torch.cat([py, base[1], oy], 1).contiguous()
        nbx, nby, nbi = col(1), col(1), zero(1)
        assert l.gecc_batch_pdbl_dev(ctx.h, C.c_size_t(1), vp(base[0]), vp(base[1]), None, vp(nbx), vp(nby), vp(nbi)) == 0
        base = (nbx, nby)
    torch.cuda.synchronize()
    # the order above is not 1..n: recover each point's multiplier the same way
    mult = np.array([1], dtype=object)
    for k in range(args.log2n - 1):
        mult = np.concatenate([mult, np.array([1 << k], dtype=object), mult + (1 << k)])
    px = torch.cat([px, px[:, :1]], 1).contiguous()   # n - 1 points so far: repeat the first
    py = torch.cat([py, py[:, :1]], 1).contiguous()
    mult = np.concatenate([mult, mult[:1]])
    assert px.shape[1] == n
    rs = np.random.RandomState(4321 + rank)
    hk = rs.randint(0, 2**32, size=(8, n), dtype=np.uint64).astype(np.uint32)
    k = torch.from_numpy(hk).cuda()
    pinf = zero(n)
    ox, oy, oi = col(1), col(1), zero(1)
    step = lambda: l.gecc_msm_dev(ctx.h, C.c_size_t(n), vp(k), vp(px), vp(py), vp(pinf), vp(ox), vp(oy), vp(oi))
    assert step() == 0
    torch.cuda.synchronize()
    ks = gecc.ints_from_cols(hk)
    total = sum((a % B.n) * int(b) for a, b in zip(ks, mult)) % B.n
    want = E.ec_mul(B, total, B.G)
    rinv = pow(R12, -1, B.p)
    got = (gecc.ints_from_cols(ox.cpu().numpy().view(np.uint32))[0] * rinv % B.p,
           gecc.ints_from_cols(oy.cpu().numpy().view(np.uint32))[0] * rinv % B.p)
    assert int(oi.item()) == 0 and got == want, "BLS MSM gate failed"

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    sctx = gecc.Context(gecc.SECP256K1, local_rank)
    peak = sctx.microbench(1, 3000)
    sctx.close()
    peak_mad_per_s = peak["total_ops"] / peak["seconds"]
    for _ in range(args.warmup):
        assert step() == 0
    barrier()
    sampler = ClockSampler(local_rank)
    launches0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        assert step() == 0
    ev1.record(stream)
    barrier()
    dev_s = ev0.elapsed_time(ev1) * 1e-3
    if world > 1:
        t = torch.tensor([dev_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t.item())
    clocks = sampler.stop()
    per = dev_s / args.steps
    counts = msm_products_per_point("generic12")
    # 12-limb Montgomery product: 144 (product) + 144 (word-serial rows m_i * q) wide multiplies + 12 m_i
    slots = {"mul_generic12": 144 + 144, "sqr_generic12": 78 + 144}   # IMAD.WIDE only
    mads = n * sum(slots[kk] * v for kk, v in counts.items())
    if rank == 0:
        print(json.dumps({
            "metric": "msm_time", "value": per * 1e3, "unit": "ms per MSM", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": f"u32 limbs ({B.p.bit_length()}-bit modular integer, 12 limbs)", "data": "synthetic",
            "config": {"workload": f"{args.curve} G1 Pippenger MSM, 2^{args.log2n} points per GPU (c = 16, batch-affine buckets)",
                       "curve": args.curve, "lanes_per_gpu": n, "sharding": f"point ranges x{world}",
                       "l2": "no L2 flush; scalars + points 2^20 x 128 B = 134 MB > 126 MB L2"},
            "clocks": clocks, "e2e": None, "gpu_launches": ctx.launches - launches0,
            "roofline": {"bound": "imad", "kernel": "k_msm_tree_fwd/bwd", "achieved": mads / per / 1e12,
                         "peak": peak_mad_per_s / 1e12, "unit": "T IMAD.WIDE-slot/s", "frac": mads / per / peak_mad_per_s,
                         "work_per_lane": {"executed": counts, "slots_per_op": slots}, "traffic": None},
            "cpu_baseline": None}), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def _ncu_traffic(wl, log2n=20):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel, per launch, from the
    committed `ncu --set full` capture of this round's kernels (profiles/r02_*, tools/ncu_summary.py);
    None when this round has no capture for the leg (stale captures are not quoted)."""
    import csv
    name, kernel = {"verify": ("r02_verify", "k_verify"), "sign": ("r02_sign", "k_sign"),
                    "padd": ("r02_padd" + ("16" if log2n <= 16 else ""), "k_"),
                    "msm": ("r02_msm", "k_msm")}.get(wl, (None, None))
    if not name:
        return None
    try:
        tot, names = 0.0, set()
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        inside = wl != "msm"   # the MSM capture is a window of launches: one MSM = k_msm_hist .. k_msm_red_final
        done = False
        with open(os.path.join(ROOT, "profiles", name + "_metrics.csv")) as f:
            for r in csv.reader(f):
                if len(r) < 4 or kernel not in r[0] or done:
                    continue
                if wl == "msm":
                    if not inside and "k_msm_hist" in r[0]:
                        inside = True
                if inside and r[1] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    tot += float(r[3]) * scale.get(r[2], 1)
                    names.add(r[0])
                    if wl == "msm" and "k_msm_red_final" in r[0] and r[1] == "dram__bytes_write.sum":
                        done = True   # the closing launch's last DRAM row (tools/ncu_summary.py keeps the report's metric order)
        return {"bytes_per_launch": tot, "kernels": sorted(names), "source": f"profiles/{name}_metrics.csv"} if tot else None
    except OSError:
        return None


def _measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


if __name__ == "__main__":
    main()
