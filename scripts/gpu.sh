#!/usr/bin/env bash
# Build the in-tree library (fails loudly), then run a command on the GPU box.
#   scripts/gpu.sh [--gpus N] [--timeout S] -- 'command'
set -euo pipefail
cd "$(dirname "$0")/.."
python -m paper_2511_16193_b200.build > /dev/null
exec /usr/local/graft/bin/gpurun "$@"
