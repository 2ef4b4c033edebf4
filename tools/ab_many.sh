#!/bin/bash
# Same-box A/B/... of library builds on the config-2 pass (tools/c2_stages.py
# medians), alternating, 2 rounds.  Usage: tools/ab_many.sh DIR1 DIR2 ... (each holding libapexb200.so)
for round in 1 2; do for v in "$@"; do APEX_B200_LIB=$PWD/$v/libapexb200.so python tools/c2_stages.py 2>/dev/null | tail -1 | sed "s|^|$v |"; done; done
