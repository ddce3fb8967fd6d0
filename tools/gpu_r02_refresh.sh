O=gpurun_out; T=r02; mkdir -p $O
(timeout 1500 python -m pytest tests -x -q -m gpu > $O/${T}_gputest.log 2>&1; echo "pytest rc $?" >> $O/${T}_gputest.log)
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 600 python bench.py --curve sm2 --workload sign > $O/${T}_bench_sm2_sign.json 2> $O/${T}_bench_sm2_sign.err
timeout 1200 bash tools/profile_r02.sh $T lists sign > $O/${T}_profile.log 2>&1
GECC_BENCH_FORCE_EXCHANGE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > $O/${T}_bench_torchrun_1rank.json 2> $O/${T}_bench_torchrun_1rank.err
(python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc $?" >> $O/${T}_smoke.log)
S=$O/${T}_sanitizer_sign.txt; : > $S
for tool in memcheck racecheck; do
  echo "== $tool: tests/test_gpu_ecdsa.py" >> $S
  timeout 1200 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_ecdsa.py -q -m gpu -k "not large and not 2p16 and not properties" 2>&1 | grep -E "passed|failed|SUMMARY|hazard|Invalid|error" | tail -6 >> $S
done
tail -3 $O/${T}_gputest.log; tail -2 $O/${T}_smoke.log; cat $S
python - <<PY
import json
d=json.loads(open('$O/${T}_bench.json').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ("metric","value","ms_per_step","gpu_launches")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
for k,v in (d.get("extra") or {}).items(): print("  ",k,v.get("value"),v.get("ms_per_step"),"frac",v.get("roofline",{}).get("frac"),"e2e",(v.get("e2e") or {}).get("value"))
PY
