#!/bin/bash
# Same-box A/B of library builds on the config-2 per-query breakdown:
#   tools/ab_perq.sh LIB...   (two rounds, interleaved)
for round in 1 2; do
  for lib in "$@"; do
    APEX_B200_LIB=$lib python tools/c2_per_query.py | sed "s|^|$(basename $lib) |"
  done
done
