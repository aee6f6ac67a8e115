#!/bin/bash
# The whole verification sequence of this repository in one place.
#   tools/verify_all.sh cpu     build + CPU suite (no GPU needed)
#   tools/verify_all.sh gpu     on a B200: GPU suite, smoke, bench lines for cfg 1-5
set -e
cd "$(dirname "$0")/.."
case "${1:-cpu}" in
  cpu)
    python -c "import __graft_entry__ as g; g.build()"
    python -m pytest tests -x -q -m "not gpu"
    ;;
  gpu)
    python -m pytest tests -x -q -m gpu
    python -c "import __graft_entry__ as g; g.smoke()"
    for c in 5 1 2 3 4; do python bench.py --config "$c"; done
    ;;
  *)
    echo "usage: tools/verify_all.sh cpu|gpu" >&2
    exit 2
    ;;
esac
