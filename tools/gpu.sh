#!/bin/bash
# Build the extension here, then run a command on the GPU box via gpurun.
#   tools/gpu.sh <timeout_s> '<command>'
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -v "Warning: The 'compute_" || true
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
