#!/bin/bash
# round-2 GPU session f: MSM window groups 1 / 2 / 4, coop padd K by size with 4 blocks per SM
O=gpurun_out; mkdir -p $O
timeout 300 python tools/exp/padd_forms.py coop128,fused 10,12,14,15,16,17,18,20 > $O/r02f_padd_forms.txt 2>&1
for g in 1 2 4; do
  GECC_MSM_GROUPS=$g timeout 300 python bench.py --workload msm --no-cpu-baseline > $O/r02f_bench_msm_g$g.json 2> $O/r02f_bench_msm_g$g.err
  GECC_MSM_GROUPS=$g timeout 300 python bench.py --workload msm --curve bls12_377 --no-cpu-baseline > $O/r02f_bench_msm_bls377_g$g.json 2> $O/r02f_bench_msm_bls377_g$g.err
done
cat $O/r02f_padd_forms.txt
for f in $O/r02f_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
