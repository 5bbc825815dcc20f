#!/bin/bash
# Variant library for A/B timing (dev tool): recompile the FAST units of the given sizes with
# extra flags on top of the default build's objects and link build_variants/NAME.so.
#   bash tools/variant.sh NAME "-DHAFB_X=1 ..." 30 32
NAME=$1; FLAGS=$2; shift 2
DEF=$(ls -d build/obj-* | head -1)
[ -n "$HAFB_DEFAULT_OBJ" ] && DEF=$HAFB_DEFAULT_OBJ
OUT=build/variant-obj-$NAME; mkdir -p $OUT
cp -u $DEF/*.o $OUT/
for S in "$@"; do
  SS=$(printf %02d $S)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -Xcompiler -O2 -I include $FLAGS -DHAFB_S=$S -Xptxas=-v \
    -c paper_1805_12498_b200/csrc/fast_inst.cu -o $OUT/fast_$SS.o 2> $OUT/fast_$SS.log &
done
wait
for S in "$@"; do SS=$(printf %02d $S); if grep -q "error" $OUT/fast_$SS.log; then echo "COMPILE FAILED for S=$S:"; grep -m3 "error" $OUT/fast_$SS.log; exit 1; fi; done
for S in "$@"; do SS=$(printf %02d $S); python tools/ptxas_regs.py "false, false, [0-9]+, false" < $OUT/fast_$SS.log; done
nvcc -gencode arch=compute_100a,code=sm_100a --shared -o build_variants/$NAME.so $OUT/*.o && echo built build_variants/$NAME.so
