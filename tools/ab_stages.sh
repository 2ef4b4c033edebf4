#!/bin/bash
# Same-box A/B of two library builds on the config-2 pass: tools/c2_stages.py
# (median of 31 graph-replayed passes, per-stage events) alternately, 3 rounds.
# Usage: tools/ab_stages.sh LIB_A LIB_B [APEX_OPTS]
A=$1; B=$2; O=${3:-}
for round in 1 2 3; do
  for lib in "$A" "$B"; do
    APEX_OPTS=$O APEX_B200_LIB=$lib python tools/c2_stages.py 2>/dev/null | tail -1 | sed "s|^|$(basename $(dirname $lib))/$(basename $lib) |"
  done
done
