#!/bin/bash
# Build in-tree, then run a command on the B200 box via gpurun (from the repo root).
#   tools/gpu.sh [--timeout S] -- '<command>'
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2212_00964_b200 import _build; _build.build(force=False)"
exec /usr/local/graft/bin/gpurun "$@"
