#!/bin/bash
# round-2 GPU session g: full parity run, default bench, reference arm, ncu evidence (summarised on the box)
O=gpurun_out; mkdir -p $O
(timeout 1500 python -m pytest tests -x -q -m gpu > $O/r02g_gputest.log 2>&1; echo "pytest rc $?" >> $O/r02g_gputest.log)
timeout 900 python bench.py > $O/r02g_bench.json 2> $O/r02g_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/r02g_bench_ref.json 2> $O/r02g_bench_ref.err
timeout 2400 bash tools/profile_r02.sh r02g lists verify sign padd padd16 msm > $O/r02g_profile.log 2>&1
tail -3 $O/r02g_gputest.log
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02g_bench.json').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ("metric","value","ms_per_step")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
for k,v in (d.get("extra") or {}).items(): print("  ",k,v.get("value"),v.get("ms_per_step"),"frac",v.get("roofline",{}).get("frac"),"e2e",(v.get("e2e") or {}).get("value"))
PY
ls -la $O | tail -30
