#!/bin/bash
# round-2 GPU session d: warp-cooperative inversion (const / var divsteps): latency, parity, effect on padd and MSM
O=gpurun_out; mkdir -p $O
timeout 120 tools/exp/_build/inv_exp > $O/r02d_inv.txt 2>&1
(timeout 1200 python -m pytest tests/test_gpu_field.py tests/test_gpu_batch.py tests/test_gpu_msm.py tests/test_gpu_bls.py tests/test_gpu_round2.py -x -q -m gpu > $O/r02d_gputest.log 2>&1; echo "pytest rc $?" >> $O/r02d_gputest.log)
timeout 300 python tools/exp/padd_forms.py chunked,coop128,fused 12,14,16,18,20 > $O/r02d_padd_forms.txt 2>&1
GECC_LIB=$PWD/paper_2501_03245_b200/lib/libgecc_b200_wvar.so timeout 300 python tools/exp/padd_forms.py chunked,coop128,fused 12,14,16,18,20 > $O/r02d_padd_forms_wvar.txt 2>&1
for form in 0 3 4; do
  GECC_MSM_FORM=$form timeout 300 python bench.py --workload msm --no-cpu-baseline > $O/r02d_bench_msm_form$form.json 2> $O/r02d_bench_msm_form$form.err
  GECC_LIB=$PWD/paper_2501_03245_b200/lib/libgecc_b200_wvar.so GECC_MSM_FORM=$form timeout 300 python bench.py --workload msm --no-cpu-baseline > $O/r02d_bench_msm_wvar_form$form.json 2> $O/r02d_bench_msm_wvar_form$form.err
done
GECC_MSM_FORM=0 timeout 300 python bench.py --workload msm --curve bls12_377 --no-cpu-baseline > $O/r02d_bench_msm_bls377.json 2> $O/r02d_bench_msm_bls377.err
tail -3 $O/r02d_gputest.log; cat $O/r02d_inv.txt; cat $O/r02d_padd_forms.txt; echo WVAR; cat $O/r02d_padd_forms_wvar.txt
for f in $O/r02d_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
