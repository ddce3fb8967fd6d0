"""world_size-2 tests of the multi-GPU host logic on CPU (gloo): lanes sharded by range
with the global lane index as nonce stream must reproduce the single-call bytes; MSM
partial sums exchanged by one all_gather must add up to the full sum.  The compute
engine injected here is the CPU checker (oracle) -- on the GPU box the same functions
drive paper_2501_03245_b200.Context (bench.py)."""
import os
import random

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import coracle as O
from oracle import pyec as E
from paper_2501_03245_b200 import shard
from tests.util import CURVE_IDS, golden

ECDSA = golden("ecdsa")


class OracleEngine:
    """Context-shaped adapter over the C oracle (test double for the GPU context)."""

    def __init__(self, cid):
        self.cid = cid

    def sign(self, dig, sec, seed, lane_base=0):
        return O.ecdsa_sign(self.cid, dig, sec, seed, lane_base=lane_base)

    def verify(self, dig, pub, sig):
        return O.ecdsa_verify(self.cid, dig, pub, sig)

    def keygen(self, seed, count, lane_base=0):
        return O.keygen(self.cid, seed, count, lane_base=lane_base)

    def msm(self, scalars, P):
        return O.msm(self.cid, scalars, P)

    def batch_padd(self, P, T):
        return O.batch_padd(self.cid, P, T)


def test_shard_range_partitions():
    for total in (0, 1, 7, 64, 1 << 20):
        for world in (1, 2, 3, 8):
            at = 0
            sizes = []
            for r in range(world):
                b, e = shard.shard_range(total, r, world)
                assert b == at and e >= b
                at = e
                sizes.append(e - b)
            assert at == total and max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.shard_range(10, 2, 2)


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ent, cid = ECDSA[name], CURVE_IDS[name]
        eng = OracleEngine(cid)
        sec, pub = bytes.fromhex(ent["secrets"]), bytes.fromhex(ent["publics"])
        dig, sig = bytes.fromhex(ent["digests"]), bytes.fromhex(ent["sigs"])
        n = ent["n"]
        ok = shard.keygen_sharded(eng, ent["keygen_seed"], n, rank, world, dist) == (0, sec, pub)
        ok &= shard.sign_sharded(eng, dig, sec, ent["nonce_seed"], rank, world, dist) == (0, sig, [0] * n)
        bad = bytearray(sig)
        bad[64 * 3 + 1] ^= 2
        bad[64 * (n - 2) + 40] ^= 2
        want = bytearray(b"\x01" * n)
        want[3] = want[n - 2] = 0
        ok &= shard.verify_sharded(eng, dig, pub, bytes(bad), rank, world, dist) == (0, bytes(want))
        # MSM: sum_i s_i * (t_i G) == (sum s_i t_i) G, computed with Python ints
        c = E.CURVES[cid]
        rng = random.Random(17)
        m = 13
        s = [rng.randrange(c.n) for _ in range(m)]
        t = [rng.randrange(1, c.n) for _ in range(m)]
        P = O.batch_fpmul(cid, O.ints_to_cols(t))
        got = shard.msm_sharded(eng, O.ints_to_cols(s), P, rank, world, dist)
        want_pt = O.batch_fpmul(cid, O.ints_to_cols([sum(a * b for a, b in zip(s, t)) % c.n]))
        ok &= all((a == b).all() for a, b in zip(got, want_pt))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["secp256k1", "sm2"])
def test_sharded_equals_single_call_gloo(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.randrange(2000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    results = dict(q.get(timeout=5) for _ in range(world))
    assert results == {0: True, 1: True}
