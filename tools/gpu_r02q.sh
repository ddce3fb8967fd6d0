#!/bin/bash
O=gpurun_out; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_msm.py tests/test_gpu_bls.py -x -q -m gpu > $O/r02q_gputest.log 2>&1; echo "pytest rc $?" >> $O/r02q_gputest.log)
for c in secp256k1 bls12_377 sm2; do
  timeout 300 python bench.py --workload msm --curve $c --no-cpu-baseline > $O/r02q_bench_msm_$c.json 2> $O/r02q_bench_msm_$c.err
done
tail -3 $O/r02q_gputest.log
for f in $O/r02q_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
