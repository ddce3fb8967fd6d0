#!/bin/bash
O=gpurun_out; mkdir -p $O
for cut in 7 8 9 10 11; do
  GECC_MSM_CUT=$cut timeout 300 python bench.py --workload msm --no-cpu-baseline > $O/r02i_bench_msm_cut$cut.json 2> $O/r02i_bench_msm_cut$cut.err
  GECC_MSM_CUT=$cut timeout 300 python bench.py --workload msm --curve bls12_377 --no-cpu-baseline > $O/r02i_bench_msm_bls377_cut$cut.json 2> $O/r02i_bench_msm_bls377_cut$cut.err
done
for f in $O/r02i_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
