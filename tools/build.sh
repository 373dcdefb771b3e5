#!/bin/sh
# rebuild the CUDA library in-tree (from any cwd)
cd "$(dirname "$0")/.." && exec python -m paper_2511_01465_b200.build "$@"
