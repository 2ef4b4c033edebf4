#!/bin/bash
# Same-box A/B of library builds over configs (tools/sweep.py, per-stage medians), 2 rounds.
# Usage: tools/ab_sweep.sh "c1 c3 c4" DIR1 DIR2 ...
CFGS=$1; shift
for r in 1 2; do for v in "$@"; do for c in $CFGS; do APEX_B200_LIB=$PWD/$v/libapexb200.so python tools/sweep.py $c - 2>/dev/null | tail -1 | sed "s|^|$v |"; done; done; done
