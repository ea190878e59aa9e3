#!/bin/bash
# A/B ncu captures of the decode kernel: 21-layer page-layer arena at tpp=16 vs tpp=32.
OUT=${1:-gpurun_out}
for T in 16 32; do
  SWEEP_TPP=$T SWEEP_LAYERS=21 SWEEP_LAYER=0 ncu --set full --clock-control none -k regex:paged_decode -s 3 -c 1 \
     -o $OUT/prof_tpp$T python profiles/sweep_decode.py --one > $OUT/ncu_tpp$T.log 2>&1
done
