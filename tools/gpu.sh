#!/bin/bash
# Build the extension here, then run a command on the GPU box via gpurun.
#   tools/gpu.sh <timeout_s> '<command>'
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /tmp/dgb_build.log 2>&1 || { grep -B2 -A6 "error" /tmp/dgb_build.log | head -60; echo "build failed"; exit 1; }
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
