#!/bin/bash
# Quick GPU check of a kernel change (dev tool): FAST parity tests, then full-step
# timing and the per-class launch list.  Usage: bash tools/gpu_quick.sh TAG
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_referee.py -x -q -m gpu > gpurun_out/tq_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/tq_$TAG.log
timeout 300 python tools/ab_time.py > gpurun_out/ab_$TAG.log 2>&1
timeout 300 python tools/ab_time.py 56 >> gpurun_out/ab_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:.*_kernel.*" --csv \
  --log-file gpurun_out/launch_$TAG.csv python tools/class_time.py fast > /dev/null 2>&1
python tools/class_eff.py gpurun_out/launch_$TAG.csv > gpurun_out/eff_$TAG.txt 2>&1
tail -3 gpurun_out/tq_$TAG.log; cat gpurun_out/ab_$TAG.log; grep -E "S=(2[2-9]|3[0-9])" gpurun_out/eff_$TAG.txt; tail -1 gpurun_out/eff_$TAG.txt
