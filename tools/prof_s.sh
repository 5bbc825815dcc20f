mkdir -p gpurun_out
for S in 28 34 22; do
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:fast_term_kernel<.int.$S," -c 1 -o gpurun_out/ncu_full_S${S}_s3 python tools/class_time.py fast > gpurun_out/ncu_S${S}.log 2>&1; echo "S$S rc=$?"
done
