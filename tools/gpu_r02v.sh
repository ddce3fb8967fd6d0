#!/bin/bash
O=gpurun_out; mkdir -p $O
for v in s2b4 s2b6; do
  GECC_LIB=$PWD/paper_2501_03245_b200/lib/libgecc_b200_$v.so timeout 300 python bench.py --curve sm2 --no-extra --no-cpu-baseline > $O/r02v_bench_sm2_verify_$v.json 2> $O/r02v_bench_sm2_verify_$v.err
done
for f in $O/r02v_bench*.json; do echo $f; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "frac", (d.get("roofline") or {}).get("frac"))
except Exception as e: print("ERR",e); print(open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
done
