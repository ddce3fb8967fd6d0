#!/bin/bash
# quick A/B on one B200: ECDSA parity tests + the verify / sign bench lines of both curves
O=gpurun_out; T=${1:-quick}; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_ecdsa.py tests/test_gpu_dev_api.py tests/test_gpu_round2.py tests/test_gpu_cpp_compat.py -x -q -m gpu > $O/${T}_gputest.log 2>&1; echo "pytest rc $?" >> $O/${T}_gputest.log)
for c in secp256k1 sm2; do
timeout 300 python bench.py --no-extra --no-cpu-baseline --curve $c > $O/${T}_bench_verify_$c.json 2> $O/${T}_bench_verify_$c.err
timeout 300 python bench.py --workload sign --no-cpu-baseline --curve $c > $O/${T}_bench_sign_$c.json 2> $O/${T}_bench_sign_$c.err
done
tail -3 $O/${T}_gputest.log
for f in $O/${T}_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
