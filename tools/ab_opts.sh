#!/bin/bash
# Same-box A/B of option sets on the config-2 pass (tools/c2_stages.py medians), 2 rounds.
# Usage: tools/ab_opts.sh "opt=v,..." "opt=v,..." ...
for r in 1 2; do for o in "$@"; do APEX_OPTS=$o python tools/c2_stages.py 2>/dev/null | tail -1; done; done
