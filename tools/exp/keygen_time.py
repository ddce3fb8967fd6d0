import time, sys
sys.path.insert(0, '.')
import paper_2501_03245_b200 as gecc
for curve in (gecc.SECP256K1, gecc.SM2):
    ctx = gecc.Context(curve, 0)
    n = 1 << 20
    for _ in range(2):
        t0 = time.perf_counter(); rc, sec, pub = ctx.keygen(7, n); t1 = time.perf_counter()
    print(curve, "keygen 2^20 host call %.2f ms" % ((t1 - t0) * 1e3))
