#!/usr/bin/env python
"""MSM size sweep: python tools/msm_sweep.py [curve ...]  ->  one JSON line per (curve, log2n)."""
import json, subprocess, sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
curves = sys.argv[1:] or ["secp256k1", "bls12_381"]
out = []
for c in curves:
    for lg in (14, 16, 18, 20, 22):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "msm", "--curve", c,
                            "--log2n", str(lg), "--steps", "5", "--warmup", "3", "--no-cpu-baseline"],
                           capture_output=True, text=True)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            out.append({"curve": c, "log2n": lg, "ms": d["ms_per_step"], "points_per_s": (1 << lg) / d["ms_per_step"] * 1e3})
            print(json.dumps(out[-1]), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"curve": c, "log2n": lg, "error": (r.stderr or str(e))[-300:]}), flush=True)
