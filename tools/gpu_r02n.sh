#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 120 tools/exp/_build/inv_exp > $O/r02n_inv.txt 2>&1
(timeout 1500 python -m pytest tests -x -q -m gpu > $O/r02n_gputest.log 2>&1; echo "pytest rc $?" >> $O/r02n_gputest.log)
timeout 300 python bench.py --no-extra --no-cpu-baseline > $O/r02n_bench_verify.json 2> $O/r02n_bench_verify.err
timeout 300 python bench.py --workload sign --no-cpu-baseline > $O/r02n_bench_sign.json 2> $O/r02n_bench_sign.err
timeout 300 python bench.py --workload padd --log2n 16 --no-cpu-baseline > $O/r02n_bench_padd16.json 2> $O/r02n_bench_padd16.err
tail -3 $O/r02n_gputest.log; head -12 $O/r02n_inv.txt
for f in $O/r02n_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
