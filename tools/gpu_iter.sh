#!/bin/bash
# One build->measure iteration on the GPU box (dev tool): GPU tests, full n=52 timing,
# per-class launch list.  Usage: bash tools/gpu_iter.sh TAG [skip-tests]
TAG=${1:-iter}
mkdir -p gpurun_out
if [ "$2" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests_$TAG.log
fi
timeout 300 python tools/quick_time.py full > gpurun_out/qt_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:.*_kernel.*" --csv \
  --log-file gpurun_out/launch_$TAG.csv python tools/class_time.py fast > /dev/null 2>&1
python tools/class_eff.py gpurun_out/launch_$TAG.csv > gpurun_out/eff_$TAG.txt 2>&1
tail -2 gpurun_out/tests_$TAG.log 2>/dev/null; cat gpurun_out/qt_$TAG.log; cat gpurun_out/eff_$TAG.txt
