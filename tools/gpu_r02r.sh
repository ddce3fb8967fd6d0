#!/bin/bash
O=gpurun_out; mkdir -p $O
for f in 0 3; do for g in 1 2 4; do
  GECC_MSM_FORM=$f GECC_MSM_GROUPS=$g timeout 300 python bench.py --workload msm --no-cpu-baseline > $O/r02r_bench_msm_f${f}_g$g.json 2> $O/r02r_bench_msm_f${f}_g$g.err
done; done
for f in $O/r02r_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
