#!/usr/bin/env python
"""Measures the integer-pipe issue rates on the GPU (roofline denominators) and
writes gpurun_out/microbench.json.  Run under gpurun."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_03245_b200 as gecc  # noqa: E402

NAMES = ["imad_wide_indep", "imad_wide_dep", "imad32", "imad_hi", "iadd3", "iadd3x_chain",
         "imad_wide+iadd_mix", "fe_mul_secp_p", "fe_mul_generic", "fe_addsub_secp_p",
         "fe_mul_secp_p_call", "fe_sqr_secp_p", "fe_sqr_secp_p_call"]


def main():
    out = {}
    with gecc.Context(gecc.SECP256K1) as ctx:
        for which, name in enumerate(NAMES):
            iters = 4000 if which < 7 else 2000
            r = ctx.microbench(which, iters)
            r["ops_per_s"] = r["total_ops"] / r["seconds"]
            r["implied_sm_mhz"] = r["ops_per_s"] / (r["ops_per_clk_per_sm"] * 148) / 1e6
            out[name] = r
            print(f"{name:22s} {r['ops_per_clk_per_sm']:8.2f} ops/clk/SM  {r['ops_per_s']/1e9:10.2f} Gops/s"
                  f"  (~{r['implied_sm_mhz']:.0f} MHz)")
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/microbench.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
