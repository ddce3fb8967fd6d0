#!/bin/bash
# round-2 GPU session e: window-group MSM pipeline, coop K by size + rotating inversion warp, lazy-field coop padd
O=gpurun_out; mkdir -p $O
(timeout 1500 python -m pytest tests -x -q -m gpu > $O/r02e_gputest.log 2>&1; echo "pytest rc $?" >> $O/r02e_gputest.log)
timeout 300 python tools/exp/padd_forms.py chunked,coop128,fused 10,12,14,16,17,18,20 > $O/r02e_padd_forms.txt 2>&1
for c in secp256k1 sm2 bls12_377 bls12_381; do
  timeout 300 python bench.py --workload msm --curve $c --no-cpu-baseline > $O/r02e_bench_msm_$c.json 2> $O/r02e_bench_msm_$c.err
done
ncu --clock-control none --metrics gpu__time_duration.sum -c 300 --csv --log-file $O/r02e_msm_launches.csv \
   python bench.py --workload msm --steps 1 --warmup 1 --no-cpu-baseline > $O/r02e_msm_lists.log 2>&1
timeout 300 python tools/msm_sweep.py > $O/r02e_msm_sweep.jsonl 2> $O/r02e_msm_sweep.err
tail -3 $O/r02e_gputest.log; cat $O/r02e_padd_forms.txt; tail -12 $O/r02e_msm_sweep.jsonl | cut -c1-200
for f in $O/r02e_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
