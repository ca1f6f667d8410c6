#!/bin/bash
# A/B of two library builds (ab/lib_base.so, ab/lib_new.so) on any command:
# bash tools/ab_cmd.sh ROUNDS command...   (the in-tree library is restored)
R=${1:-3}; shift
L=paper_2510_19764_b200/libsparsewire_b200.so
cp $L /tmp/lib_keep.so
for i in $(seq $R); do
  for v in base new; do
    cp ab/lib_$v.so $L
    echo "== $v"; "$@"
  done
done
cp /tmp/lib_keep.so $L
