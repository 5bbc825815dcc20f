set -x
python tools/prof_fast.py 1 > gpurun_out/prof_plain.log 2>&1 || exit 1
for S in 28 34 22; do
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:fast_term_kernel<.int.$S," -c 1 -o gpurun_out/ncu_S$S python tools/prof_fast.py 1 > gpurun_out/ncu_S$S.log 2>&1
done
ls -la gpurun_out
