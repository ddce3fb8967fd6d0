#!/bin/bash
# Round-2 evidence run (one B200, under gpurun): launch lists of the bench command and one
# `ncu --set full` capture per hot kernel.  Outputs land in gpurun_out/; tools/ncu_summary.py
# turns each .ncu-rep into profiles/<tag>_{metrics,opmix}.csv here.
#   usage: tools/profile_r02.sh <tag> [legs...]      legs: verify sign padd padd16 msm lists
set -u
TAG=${1:-r02}; shift || true
LEGS=${*:-"lists verify sign padd padd16 msm"}
OUT=gpurun_out
mkdir -p $OUT
NCU="ncu --clock-control none"
for leg in $LEGS; do
  case $leg in
    lists)
      $NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $OUT/${TAG}_launches.csv \
        python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/${TAG}_lists.log 2>&1 ;;
    verify)
      $NCU --set full --import-source on -k regex:k_verify -s 3 -c 1 -f -o $OUT/${TAG}_verify \
        python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > $OUT/${TAG}_verify.log 2>&1 ;;
    sign)
      $NCU --set full --import-source on -k regex:k_sign -s 3 -c 1 -f -o $OUT/${TAG}_sign \
        python bench.py --workload sign --steps 2 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_sign.log 2>&1 ;;
    padd)
      $NCU --set full --import-source on -k regex:'k_batch_padd|k_padd' -s 4 -c 4 -f -o $OUT/${TAG}_padd \
        python bench.py --workload padd --steps 2 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_padd.log 2>&1 ;;
    padd16)
      $NCU --set full --import-source on -k regex:'k_batch_padd|k_padd' -s 4 -c 1 -f -o $OUT/${TAG}_padd16 \
        python bench.py --workload padd --log2n 16 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_padd16.log 2>&1 ;;
    msm)
      $NCU --set full --import-source on -k regex:k_msm -s 60 -c 60 -f -o $OUT/${TAG}_msm \
        python bench.py --workload msm --steps 1 --warmup 1 --no-cpu-baseline > $OUT/${TAG}_msm.log 2>&1 ;;
  esac
done
# the .ncu-rep files (source imported) are far beyond what gpurun brings back (64 MiB for the whole
# directory): summarise them ON the box and keep only the CSVs
for rep in $OUT/${TAG}_*.ncu-rep; do
  [ -f "$rep" ] || continue
  python tools/ncu_summary.py "$rep" "${rep%.ncu-rep}" > /dev/null 2>&1
  rm -f "$rep"
done
ls -la $OUT | tail -30
