"""Multi-GPU sharding of the batch path: one process per GPU (torchrun), lanes are
split into contiguous ranges, no data-path collective.

* ECDSA sign / verify / keygen / ECDH and the batch point kernels are independent
  per lane: rank r processes lanes [begin_r, end_r) on its own GPU and
  passes ``lane_base = begin_r`` so that the nonce stream id stays the *global* lane
  index (reference: protocol.cpp:125-126) -- the bytes equal a single-GPU call.
* MSM shards by point range; every rank produces one partial sum and the partial
  sums are exchanged with ONE small all_gather (65 bytes per rank) and added locally
  (EC addition is not a reduction operator NCCL knows).

``engine`` is anything with the Context method signatures (the GPU Context in
production; the tests inject a CPU checker so the host logic runs under gloo).
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Balanced contiguous ranges, sizes differ by at most one (LanePlan::make,
    batch_invert.cpp:8-29, applied to ranks instead of lanes)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    base, rem = divmod(total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def _gather_bytes(local: bytes, dist, world: int) -> List[bytes]:
    if world == 1:
        return [local]
    out: List = [None] * world
    dist.all_gather_object(out, local)
    return out


def sign_sharded(engine, digests: bytes, secrets: bytes, nonce_seed: int, rank: int, world: int,
                 dist=None):
    """Every rank passes the full inputs (or at least its slice) and gets the full result."""
    n = len(digests) // 32
    b, e = shard_range(n, rank, world)
    rc, sig, st = engine.sign(digests[32 * b:32 * e], secrets[32 * b:32 * e], nonce_seed, lane_base=b)
    parts = _gather_bytes((rc, sig, st), dist, world)
    rcs = [p[0] for p in parts]
    first_bad = next((r for r in rcs if r != 0), 0)
    if first_bad:   # a failed rank returned no usable slice: joining would misalign the lanes
        return first_bad, b"", []
    return 0, b"".join(p[1] for p in parts), sum((p[2] for p in parts), [])


def verify_sharded(engine, digests: bytes, publics: bytes, sigs: bytes, rank: int, world: int,
                   dist=None):
    n = len(digests) // 32
    b, e = shard_range(n, rank, world)
    rc, res = engine.verify(digests[32 * b:32 * e], publics[65 * b:65 * e], sigs[64 * b:64 * e])
    parts = _gather_bytes((rc, res), dist, world)
    bad = next((p[0] for p in parts if p[0] != 0), 0)
    return bad, (b"" if bad else b"".join(p[1] for p in parts))


def keygen_sharded(engine, seed: int, count: int, rank: int, world: int, dist=None):
    b, e = shard_range(count, rank, world)
    rc, sec, pub = engine.keygen(seed, e - b, lane_base=b)
    parts = _gather_bytes((rc, sec, pub), dist, world)
    bad = next((p[0] for p in parts if p[0] != 0), 0)
    if bad:
        return bad, b"", b""
    return 0, b"".join(p[1] for p in parts), b"".join(p[2] for p in parts)


def msm_sharded(engine, scalars: np.ndarray, points: Sequence[np.ndarray], rank: int, world: int,
                dist=None, add_points: Callable | None = None):
    """scalars (8, n), points = (x, y, inf).  Returns the full sum on every rank.
    ``add_points(list_of_partial_points)`` folds the gathered partial sums; by default the
    engine's own batch_padd is used (log2(world) calls on one-element batches)."""
    n = scalars.shape[1]
    b, e = shard_range(n, rank, world)
    cut = lambda a: np.ascontiguousarray(a[..., b:e])
    part = engine.msm(cut(scalars), tuple(cut(a) for a in points))
    payload = tuple(np.ascontiguousarray(a).tobytes() for a in part)
    parts = _gather_bytes(payload, dist, world)
    # limbs per coordinate follow the payload: 8 on the 256-bit curves, 12 on BLS12-381 / BLS12-377
    pts = [(np.frombuffer(p[0], np.uint32).reshape(len(p[0]) // 4, 1).copy(),
            np.frombuffer(p[1], np.uint32).reshape(len(p[1]) // 4, 1).copy(),
            np.frombuffer(p[2], np.uint8).copy()) for p in parts]
    if add_points is not None:
        return add_points(pts)
    acc = pts[0]
    for p in pts[1:]:
        acc = engine.batch_padd(acc, p)
    return acc
