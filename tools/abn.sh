#!/bin/bash
# Same-box comparison of several library builds: tools/abn.sh "LIB1 LIB2 ..." CONFIG...
LIBS=$1; shift
for round in 1 2; do
  for c in "$@"; do
    for lib in $LIBS; do
      APEX_B200_LIB=$lib python tools/sweep.py $c - | sed "s|^|$(basename $lib) |"
    done
  done
done
