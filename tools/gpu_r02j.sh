#!/bin/bash
O=gpurun_out; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_ecdsa.py tests/test_gpu_dev_api.py tests/test_gpu_round2.py -x -q -m gpu > $O/r02j_gputest.log 2>&1; echo "pytest rc $?" >> $O/r02j_gputest.log)
timeout 300 python bench.py --no-extra --no-cpu-baseline > $O/r02j_bench_verify.json 2> $O/r02j_bench_verify.err
timeout 300 python bench.py --no-extra --no-cpu-baseline --curve sm2 > $O/r02j_bench_verify_sm2.json 2> $O/r02j_bench_verify_sm2.err
tail -3 $O/r02j_gputest.log
for f in $O/r02j_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
