#!/usr/bin/env bash
# Rebuild the library with device-side bounds asserts (-DSR_DEBUG_CHECKS) and
# run the GPU test suite against it, then restore the release build.
# compute-sanitizer is closed on the GPU pool, so this is the memory-safety
# pass of the hot path (every index computed from device state is asserted).
set -euo pipefail
cd "$(dirname "$0")/.."
SR_EXTRA_NVCC_FLAGS=-DSR_DEBUG_CHECKS python -m paper_2511_16193_b200.build
python -m pytest tests -m gpu -q -x "$@"
python -m paper_2511_16193_b200.build
