#!/bin/bash
# Same-box A/B of two builds of the library: tools/ab.sh LIB_A LIB_B CONFIG...
A=$1; B=$2; shift 2
for round in 1 2; do
  for c in "$@"; do
    for lib in "$A" "$B"; do
      APEX_B200_LIB=$lib python tools/sweep.py $c - | sed "s|^|$(basename $lib) |"
    done
  done
done
