#!/bin/bash
# round-2 GPU session h: parity run with the runtime-modulus layer + padd captures
O=gpurun_out; mkdir -p $O
(timeout 1500 python -m pytest tests -x -q -m gpu > $O/r02h_gputest.log 2>&1; echo "pytest rc $?" >> $O/r02h_gputest.log)
timeout 1200 bash tools/profile_r02.sh r02h padd padd16 > $O/r02h_profile.log 2>&1
tail -15 $O/r02h_gputest.log
