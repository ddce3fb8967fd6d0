#!/bin/bash
# Round-2 evidence run on one B200 (under gpurun): parity suite, bench lines of every leg and curve, the
# reference arm, launch lists + ncu captures (summarised on the box), sweeps with per-size parity
# gates, compute-sanitizer.  Everything lands in gpurun_out/ as r02_*; copy what is judged to profiles/.
O=gpurun_out; T=${1:-r02}; mkdir -p $O
(timeout 1500 python -m pytest tests -x -q -m gpu > $O/${T}_gputest.log 2>&1; echo "pytest rc $?" >> $O/${T}_gputest.log)
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/${T}_bench_reference_arm.json 2> $O/${T}_bench_reference_arm.err
for c in sm2; do
  timeout 600 python bench.py --curve $c --no-extra > $O/${T}_bench_${c}_verify.json 2> $O/${T}_bench_${c}_verify.err
  timeout 600 python bench.py --curve $c --workload sign > $O/${T}_bench_${c}_sign.json 2> $O/${T}_bench_${c}_sign.err
done
for c in sm2 bls12_381 bls12_377; do
  timeout 600 python bench.py --curve $c --workload msm --no-cpu-baseline > $O/${T}_bench_msm_$c.json 2> $O/${T}_bench_msm_$c.err
done
timeout 2400 bash tools/profile_r02.sh $T lists verify sign padd padd16 msm > $O/${T}_profile.log 2>&1
timeout 900 python tools/sweep.py > $O/${T}_sweep.log 2>&1; mv $O/sweep.json $O/${T}_sweep.json 2>/dev/null
timeout 600 python tools/msm_sweep.py secp256k1 bls12_377 > $O/${T}_msm_sweep.jsonl 2> $O/${T}_msm_sweep.err
timeout 120 tools/exp/_build/inv_exp > $O/${T}_inversion_latency.txt 2>&1
timeout 120 tools/exp/_build/padd_timeline > $O/${T}_padd16_timeline.txt 2>&1
# the launch the driver uses for N > 1, with one rank: torchrun rendezvous, NCCL init, the MSM exchange path
GECC_BENCH_FORCE_EXCHANGE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > $O/${T}_bench_torchrun_1rank.json 2> $O/${T}_bench_torchrun_1rank.err
(python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc $?" >> $O/${T}_smoke.log)
timeout 300 python tools/exp/padd_forms.py chunked,coop128,fused 10,12,14,16,18,20,22 > $O/${T}_padd_forms.txt 2>&1
# compute-sanitizer over the kernels that changed this round (shared-memory slots, warp-cooperative inversion, MSM groups)
S=$O/${T}_sanitizer.txt; : > $S
for tool in memcheck racecheck synccheck; do
  echo "== $tool: tests/test_gpu_ecdsa.py tests/test_gpu_batch.py tests/test_gpu_field.py tests/test_runtime_field.py" >> $S
  timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_ecdsa.py tests/test_gpu_batch.py tests/test_gpu_field.py tests/test_runtime_field.py -q -m gpu -k "not large and not 2p16 and not properties" 2>&1 | grep -E "passed|failed|SUMMARY|hazard|Invalid|error" | tail -6 >> $S
done
for tool in memcheck initcheck racecheck; do
  echo "== $tool: tests/test_gpu_msm.py tests/test_gpu_bls.py -k 'small or skewed or msm_g1'" >> $S
  timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_msm.py tests/test_gpu_bls.py -q -m gpu -k "small or skewed or msm_g1" 2>&1 | grep -E "passed|failed|SUMMARY|hazard|Invalid|error" | tail -6 >> $S
done
tail -3 $O/${T}_gputest.log; tail -2 $O/${T}_smoke.log; tail -c 400 $O/${T}_bench_torchrun_1rank.json; cat $S; tail -12 $O/${T}_sweep.log
python - <<PY
import json
d=json.loads(open('$O/${T}_bench.json').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ("metric","value","ms_per_step","gpu_launches")}, "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
for k,v in (d.get("extra") or {}).items(): print("  ",k,v.get("value"),v.get("ms_per_step"),"frac",v.get("roofline",{}).get("frac"),"e2e",(v.get("e2e") or {}).get("value"))
PY
ls -la $O | tail -50
