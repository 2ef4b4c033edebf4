#!/bin/bash
# build here first (nvcc cross-compiles); only ship to the GPU box if it builds
set -e
cd /root/repo
python -c "import __graft_entry__ as g; g.build()"
timeout $(( ${GPU_TIMEOUT:-1500} + 1200 )) /usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-1500} -- "$@"
