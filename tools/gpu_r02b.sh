#!/bin/bash
# round-2 GPU session b: inversion latency, tests, padd forms, bench A/B
O=gpurun_out; mkdir -p $O
timeout 120 tools/exp/_build/inv_exp > $O/r02b_inv.txt 2>&1
(timeout 1200 python -m pytest tests -m gpu -x -q > $O/r02b_gputest.log 2>&1; echo "pytest rc $?" >> $O/r02b_gputest.log)
timeout 300 python tools/exp/padd_forms.py chunked,coop128,fused 12,14,16,18,20 > $O/r02b_padd_forms.txt 2>&1
timeout 600 python bench.py > $O/r02b_bench.json 2> $O/r02b_bench.err
GECC_LIB=$PWD/paper_2501_03245_b200/lib/libgecc_b200_smem.so timeout 300 python bench.py --no-extra --no-cpu-baseline > $O/r02b_bench_smem.json 2> $O/r02b_bench_smem.err
GECC_MSM_FORM=3 timeout 300 python bench.py --workload msm --no-cpu-baseline > $O/r02b_bench_msm_form3.json 2> $O/r02b_bench_msm_form3.err
timeout 300 python bench.py --workload msm --no-cpu-baseline > $O/r02b_bench_msm.json 2> $O/r02b_bench_msm.err
timeout 300 python bench.py --workload msm --curve bls12_377 --no-cpu-baseline > $O/r02b_bench_msm_bls377.json 2> $O/r02b_bench_msm_bls377.err
GECC_MSM_FORM=3 timeout 300 python bench.py --workload msm --curve bls12_377 --no-cpu-baseline > $O/r02b_bench_msm_bls377_form3.json 2> $O/r02b_bench_msm_bls377_form3.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/r02b_bench_ref.json 2>&1
tail -3 $O/r02b_gputest.log; cat $O/r02b_inv.txt; cat $O/r02b_padd_forms.txt
for f in $O/r02b_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", d.get("e2e",{}).get("value"), "frac", d.get("roofline",{}).get("frac"))
    for k,v in (d.get("extra") or {}).items(): print("  ",k,v.get("value"),v.get("ms_per_step"),"frac",v.get("roofline",{}).get("frac"))
except Exception as e: print("ERR",e)
PY
done
