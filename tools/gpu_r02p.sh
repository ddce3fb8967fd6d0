#!/bin/bash
O=gpurun_out; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_ecdsa.py tests/test_gpu_dev_api.py tests/test_gpu_round2.py tests/test_gpu_batch.py -x -q -m gpu > $O/r02p_gputest.log 2>&1; echo "pytest rc $?" >> $O/r02p_gputest.log)
for u in 0 1 2 3 4; do
  GECC_MSM_UPPER=$u timeout 300 python bench.py --workload msm --no-cpu-baseline > $O/r02p_bench_msm_u$u.json 2> $O/r02p_bench_msm_u$u.err
  GECC_MSM_UPPER=$u timeout 300 python bench.py --workload msm --curve bls12_377 --no-cpu-baseline > $O/r02p_bench_msm_bls377_u$u.json 2> $O/r02p_bench_msm_bls377_u$u.err
done
GECC_MSM_UPPER=2 timeout 600 python -m pytest tests/test_gpu_msm.py tests/test_gpu_bls.py -x -q -m gpu -k "affine and not affine1" > $O/r02p_gputest_msm_u2.log 2>&1
tail -3 $O/r02p_gputest.log; tail -3 $O/r02p_gputest_msm_u2.log
for f in $O/r02p_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
