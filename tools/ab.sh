#!/bin/bash
# A/B of two builds of the library on one box: bash tools/ab.sh ROUNDS [bench args...]
# (ab/lib_base.so, ab/lib_new.so; the in-tree library is restored at the end)
R=${1:-3}; shift
L=paper_2510_19764_b200/libsparsewire_b200.so
cp $L /tmp/lib_keep.so
for i in $(seq $R); do
  for v in base new; do
    cp ab/lib_$v.so $L
    python bench.py --no-micro --no-cpu-baseline "$@" > /tmp/ab.json 2>/dev/null
    python tools/bench_line.py /tmp/ab.json $v
  done
done
cp /tmp/lib_keep.so $L
