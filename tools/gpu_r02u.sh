#!/bin/bash
O=gpurun_out; mkdir -p $O
(timeout 1500 python -m pytest tests -x -q -m gpu > $O/r02u_gputest.log 2>&1; echo "pytest rc $?" >> $O/r02u_gputest.log)
timeout 300 python bench.py --curve sm2 --no-extra --no-cpu-baseline > $O/r02u_bench_sm2_verify.json 2> $O/r02u_bench_sm2_verify.err
timeout 300 python bench.py --curve sm2 --workload sign --no-cpu-baseline > $O/r02u_bench_sm2_sign.json 2> $O/r02u_bench_sm2_sign.err
timeout 300 python bench.py --curve sm2 --workload msm --no-cpu-baseline > $O/r02u_bench_sm2_msm.json 2> $O/r02u_bench_sm2_msm.err
timeout 300 python bench.py --curve sm2 --workload padd --no-cpu-baseline > $O/r02u_bench_sm2_padd.json 2> $O/r02u_bench_sm2_padd.err
tail -3 $O/r02u_gputest.log
for f in $O/r02u_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
