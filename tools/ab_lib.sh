#!/usr/bin/env bash
# A/B two builds of the library on the same box: alternating processes per shape.
# usage: tools/ab_lib.sh libA.so libB.so [shape ...]
A=$1; B=$2; shift 2
shapes=${@:-4096x11008 11008x4096 8192x22016}
for s in $shapes; do
  for rep in 1 2; do
    for L in $A $B; do
      echo -n "$(basename $L) "
      QLRT_LIB_PATH=$L python tools/ab.py X=0 --shape $s --rounds 3 | sed 's/^X=0 *//'
    done
  done
done
