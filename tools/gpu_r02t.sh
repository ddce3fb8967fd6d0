#!/bin/bash
O=gpurun_out; mkdir -p $O
for k in 0 1; do
  GECC_MSM_SCATTER=$k timeout 300 python bench.py --workload msm --no-cpu-baseline > $O/r02t_bench_msm_s$k.json 2> $O/r02t_bench_msm_s$k.err
  GECC_MSM_SCATTER=$k ncu --clock-control none --metrics gpu__time_duration.sum -k regex:'k_msm_(hist|scatter|scan)' -c 40 --csv --log-file $O/r02t_sort_s$k.csv python bench.py --workload msm --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  grep -E "k_msm_(hist|scatter)" $O/r02t_sort_s$k.csv | tail -4 | cut -d, -f5,15- | cut -c1-160
done
GECC_MSM_SCATTER=1 timeout 600 python -m pytest tests/test_gpu_msm.py -x -q -m gpu -k "small or skewed" 2>&1 | tail -2
for f in $O/r02t_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value")}, "e2e", (d.get("e2e") or {}).get("value"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
