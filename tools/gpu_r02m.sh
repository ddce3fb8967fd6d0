#!/bin/bash
O=gpurun_out; mkdir -p $O
for v in sb5 sb6; do
 for c in secp256k1 sm2; do
  GECC_LIB=$PWD/paper_2501_03245_b200/lib/libgecc_b200_$v.so timeout 300 python bench.py --workload sign --no-cpu-baseline --curve $c > $O/r02m_bench_sign_${c}_$v.json 2> $O/r02m_bench_sign_${c}_$v.err
 done
done
for f in $O/r02m_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
