#!/bin/bash
# Measurement pass for profiles/ (dev tool): bench line, bench launch list, per-class
# DRAM bytes of one full step, one full ncu capture of the top class kernel.
TAG=${1:-v9}
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k "regex:fast_term_kernel" --csv --log-file gpurun_out/dram_$TAG.csv python tools/class_time.py fast > /dev/null 2>&1; echo "dram rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:fast_term_kernel<.int.28," -c 1 -o gpurun_out/ncu_full_S28_$TAG python tools/class_time.py fast > /dev/null 2>&1; echo "full rc=$?"
timeout 600 python bench.py --n 56 --steps 2 --warmup 3 --mirror-steps 0 > gpurun_out/bench_n56_$TAG.log 2>&1; echo "n56 rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
