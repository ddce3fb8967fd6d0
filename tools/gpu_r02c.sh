#!/bin/bash
# round-2 GPU session c: scheduled inversion latency, fused MSM tree parity + timing, MSM launch list
O=gpurun_out; mkdir -p $O
timeout 120 tools/exp/_build/inv_exp > $O/r02c_inv.txt 2>&1
(timeout 1200 python -m pytest tests/test_gpu_msm.py tests/test_gpu_bls.py -x -q -m gpu > $O/r02c_gputest_msm.log 2>&1; echo "pytest rc $?" >> $O/r02c_gputest_msm.log)
for form in 0 4 5; do
  GECC_MSM_FORM=$form timeout 300 python bench.py --workload msm --no-cpu-baseline > $O/r02c_bench_msm_form$form.json 2> $O/r02c_bench_msm_form$form.err
  GECC_MSM_FORM=$form timeout 300 python bench.py --workload msm --curve bls12_377 --no-cpu-baseline > $O/r02c_bench_msm_bls377_form$form.json 2> $O/r02c_bench_msm_bls377_form$form.err
done
for form in 0 4; do
ncu --clock-control none --metrics gpu__time_duration.sum -c 300 --csv --log-file $O/r02c_msm_form${form}_launches.csv \
   env GECC_MSM_FORM=$form python bench.py --workload msm --steps 1 --warmup 1 --no-cpu-baseline > $O/r02c_msm_lists$form.log 2>&1
done
tail -3 $O/r02c_gputest_msm.log; cat $O/r02c_inv.txt
for f in $O/r02c_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
